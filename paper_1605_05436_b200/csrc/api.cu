// C-ABI of libxsum.so (declared and documented in include/xsum.h).
// Host-side argument checking, handle bookkeeping and launches; every arithmetic step of
// the summation runs in the kernels (accumulate.cu, merge_finalize.cu, segments.cu).
#include <cuda_runtime.h>
#include <cstring>

#include <atomic>
#include <cstdlib>
#include <new>

#include "xsum.h"
#include "xsum_kernels.h"

static std::atomic<uint64_t> g_launches{0};

namespace xs {
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("XSUM_NO_PDL");
        return !(e && e[0] == '1');
    }();
    return on;
}
}  // namespace xs

struct xsum_ctx {
    int device;
    int num_sms;
    xsum_state_image* state;
    uint8_t* scratch;
    uint64_t count;                 // host-side mirror of the summand count (capacity check); while
                                    // count_pending: the summands added since the last merge
    bool count_pending;             // a merge changed the device count; *count_pinned holds it once
                                    // ev_count completes
    uint64_t* count_pinned;         // pinned host word (lazily allocated at the first merge)
    cudaEvent_t ev_count;
    uint32_t grid_limit;            // 0 = one block per SM
    cudaStream_t copy_stream;       // host-buffer path only (lazily created)
    cudaEvent_t ev_ready[2], ev_done[2];
};

namespace {

constexpr uint64_t kMaxCount = 0x7FFFFFFFFFFFFFFFull;

struct DeviceGuard {   // run on the handle's device, restore the caller's afterwards
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) { ok = false; return; }
        if (prev != dev && cudaSetDevice(dev) != cudaSuccess) ok = false;
    }
    ~DeviceGuard() {
        int cur;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

xs::AccParams acc_params(xsum_ctx* h, int overwrite, xsum_result* res, uint64_t* canon) {
    xs::AccParams p;
    p.state = h->state;
    p.counter = reinterpret_cast<uint32_t*>(h->scratch + xs::SCRATCH_COUNTER_OFF);
    p.gflags = reinterpret_cast<uint32_t*>(h->scratch + xs::SCRATCH_GFLAGS_OFF);
    p.gacc = reinterpret_cast<int64_t*>(h->scratch + xs::SCRATCH_ACC_OFF);
    p.stamps = XS_TIMING ? reinterpret_cast<int64_t*>(h->scratch + xs::SCRATCH_STAMP_OFF) : nullptr;
    p.overwrite = overwrite;
    p.res = res;
    p.canon = canon;
    p.one = 1;
    p.mone = 0xFFFFFFFFu;
    p.peer.bufs = nullptr;
    p.peer.rank = p.peer.world = 0;
    p.peer.epoch = 0;
    p.skip = nullptr;
    return p;
}

int grid_of(const xsum_ctx* h) {
    return h->grid_limit ? (int)(h->grid_limit < XS_MAXB ? h->grid_limit : XS_MAXB) : h->num_sms;
}

int sms_of(int dev) {
    static int cache[64] = {0};
    if (dev < 0 || dev >= 64) return 148;
    if (!cache[dev]) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        cache[dev] = v;
    }
    return cache[dev];
}

bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

// After a merge the device state's count is the merged total, unknown to the host until the
// stream gets there: enqueue a copy of it into a pinned word and remember the event; later
// accumulates add to h->count (the summands since the merge), which xsum_count adds to the
// copied word. Until then the host capacity check sees only a lower bound; the kernels saturate
// the count and set XSUM_F_CAPACITY if the true total passes 2^63-1 (count_add).
xsum_status note_merge(xsum_ctx* h, cudaStream_t s) {
    if (!h->count_pinned) {
        if (cudaHostAlloc(reinterpret_cast<void**>(&h->count_pinned), sizeof(uint64_t), cudaHostAllocDefault) !=
            cudaSuccess) {
            h->count_pinned = nullptr;
            return XSUM_ECUDA;
        }
        if (cudaEventCreateWithFlags(&h->ev_count, cudaEventDisableTiming) != cudaSuccess) {
            cudaFreeHost(h->count_pinned);
            h->count_pinned = nullptr;
            return XSUM_ECUDA;
        }
    }
    if (cudaMemcpyAsync(h->count_pinned, &h->state->count, sizeof(uint64_t), cudaMemcpyDeviceToHost, s) !=
            cudaSuccess ||
        cudaEventRecord(h->ev_count, s) != cudaSuccess)
        return XSUM_ECUDA;
    h->count_pending = true;
    h->count = 0;
    return XSUM_OK;
}

// 16-bit inputs: one launch per 2^40 summands (the kernel's int64 bin totals stay < 2^63).
xsum_status run_h16(xsum_ctx* h, const uint16_t* d_x, uint64_t n, int bf16, int overwrite, xsum_result* res,
                    uint64_t* canon, cudaStream_t s) {
    constexpr uint64_t CH = 1ull << 40;
    uint64_t off = 0;
    bool first = true;
    do {
        const uint64_t c = (n - off) < CH ? (n - off) : CH;
        const bool last = off + c == n;
        if (xs::accumulate_h16(d_x + off, c, bf16, acc_params(h, first ? overwrite : 0, last ? res : nullptr,
                                                               last ? canon : nullptr),
                               grid_of(h), s) != cudaSuccess)
            return XSUM_ECUDA;
        off += c;
        first = false;
    } while (off < n);
    return XSUM_OK;
}

xsum_status accumulate_h16_api(xsum_ctx* h, const uint16_t* d_x, uint64_t n, int bf16, void* stream) {
    if (!h) return XSUM_EINVAL;
    if (n == 0) return XSUM_OK;
    if (!d_x || !aligned(d_x, 2)) return XSUM_EINVAL;
    if (n > kMaxCount - h->count) return XSUM_ECAPACITY;
    DeviceGuard g(h->device);
    if (!g.ok) return XSUM_ECUDA;
    xsum_status st = run_h16(h, d_x, n, bf16, 0, nullptr, nullptr, static_cast<cudaStream_t>(stream));
    if (st == XSUM_OK) h->count += n;
    return st;
}

xsum_status sum_h16_api(xsum_ctx* h, const uint16_t* d_x, uint64_t n, int bf16, void* d_res, uint64_t* d_canon,
                        void* stream) {
    if (!h || !d_res || !aligned(d_res, 8) || (d_canon && !aligned(d_canon, 8))) return XSUM_EINVAL;
    if (n && (!d_x || !aligned(d_x, 2))) return XSUM_EINVAL;
    if (n > kMaxCount) return XSUM_ECAPACITY;
    DeviceGuard g(h->device);
    if (!g.ok) return XSUM_ECUDA;
    xsum_status st = run_h16(h, d_x, n, bf16, 1, static_cast<xsum_result*>(d_res), d_canon,
                             static_cast<cudaStream_t>(stream));
    if (st == XSUM_OK) {
        h->count = n;
        h->count_pending = false;
    }
    return st;
}

}  // namespace

extern "C" {

size_t xsum_state_bytes(void) { return XSUM_STATE_BYTES; }
size_t xsum_scratch_bytes(int device) { (void)device; return xs::SCRATCH_BYTES; }
size_t xsum_result_bytes(void) { return sizeof(xsum_result); }
uint64_t xsum_launch_count(void) { return g_launches.load(); }

const char* xsum_status_str(xsum_status s) {
    switch (s) {
        case XSUM_OK: return "ok";
        case XSUM_EINVAL: return "invalid argument";
        case XSUM_ECAPACITY: return "capacity exceeded (more than 2^63-1 summands)";
        case XSUM_ECUDA: return "CUDA error";
        case XSUM_EMISMATCH: return "state image mismatch";
        case XSUM_ENOMEM: return "out of host memory";
    }
    return "unknown status";
}

xsum_status xsum_create(xsum_ctx** h, int device, void* d_state, void* d_scratch, size_t scratch_bytes,
                        void* stream) {
    if (!h) return XSUM_EINVAL;
    *h = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess) return XSUM_ECUDA;
    if (device < 0 || device >= ndev) return XSUM_EINVAL;
    if (!d_state || !d_scratch || !aligned(d_state, 8) || !aligned(d_scratch, 256)) return XSUM_EINVAL;
    if (scratch_bytes < xs::SCRATCH_BYTES) return XSUM_EINVAL;
    DeviceGuard g(device);
    if (!g.ok) return XSUM_ECUDA;
    xsum_ctx* c = new (std::nothrow) xsum_ctx();
    if (!c) return XSUM_ENOMEM;
    c->device = device;
    c->num_sms = sms_of(device);
    c->state = static_cast<xsum_state_image*>(d_state);
    c->scratch = static_cast<uint8_t*>(d_scratch);
    c->count = 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(c->scratch, 0, xs::SCRATCH_BYTES, s) != cudaSuccess ||
        xs::init_state(c->state, s) != cudaSuccess) {
        delete c;
        return XSUM_ECUDA;
    }
    *h = c;
    return XSUM_OK;
}

xsum_status xsum_reset(xsum_ctx* h, void* stream) {
    if (!h) return XSUM_EINVAL;
    DeviceGuard g(h->device);
    if (!g.ok) return XSUM_ECUDA;
    if (xs::init_state(h->state, static_cast<cudaStream_t>(stream)) != cudaSuccess) return XSUM_ECUDA;
    h->count = 0;
    h->count_pending = false;
    return XSUM_OK;
}

// Checkpoint / resume: the 384-byte state image is the checkpoint.
xsum_status xsum_save_state(xsum_ctx* h, void* host_image, void* stream) {
    if (!h || !host_image) return XSUM_EINVAL;
    DeviceGuard g(h->device);
    if (!g.ok) return XSUM_ECUDA;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (cudaMemcpyAsync(host_image, h->state, XSUM_STATE_BYTES, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return XSUM_ECUDA;
    return XSUM_OK;
}

xsum_status xsum_check_state_image(const void* host_image) {
    if (!host_image) return XSUM_EINVAL;
    xsum_state_image im;
    std::memcpy(&im, host_image, sizeof im);
    if (im.magic != XSUM_MAGIC || im.version != XSUM_VERSION || im.w != 52 || im.ndigits != XSUM_NDIGITS ||
        im.reserved != 0 || (im.flags & ~(XSUM_F_NAN | XSUM_F_PINF | XSUM_F_NINF | XSUM_F_MISMATCH)) ||
        im.count > kMaxCount)
        return XSUM_EMISMATCH;
    for (unsigned char b : im.pad)
        if (b) return XSUM_EMISMATCH;
    const int64_t rmax = (1ll << 52) - 1;                 // regularized: |digit| <= R-1 (Lemma 1)
    for (int j = 0; j < XSUM_NDIGITS - 1; ++j)
        if (im.digit[j] > rmax || im.digit[j] < -rmax) return XSUM_EMISMATCH;
    // top digit (R^41 = 2^2132): |A| < 2^(1024+1074+63) bounds it by 2^29
    if (im.digit[XSUM_NDIGITS - 1] > XSUM_TOP_DIGIT_MAX || im.digit[XSUM_NDIGITS - 1] < -XSUM_TOP_DIGIT_MAX)
        return XSUM_EMISMATCH;
    return XSUM_OK;
}

xsum_status xsum_load_state(xsum_ctx* h, const void* host_image, void* stream) {
    if (!h || !host_image) return XSUM_EINVAL;
    if (xsum_status st = xsum_check_state_image(host_image)) return st;
    DeviceGuard g(h->device);
    if (!g.ok) return XSUM_ECUDA;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // pageable source: the copy is staged before the call returns, so the caller may free it
    if (cudaMemcpyAsync(h->state, host_image, XSUM_STATE_BYTES, cudaMemcpyHostToDevice, s) != cudaSuccess)
        return XSUM_ECUDA;
    uint64_t cnt;
    std::memcpy(&cnt, static_cast<const uint8_t*>(host_image) + 16, sizeof cnt);
    h->count = cnt;
    h->count_pending = false;
    return XSUM_OK;
}

xsum_status xsum_accumulate(xsum_ctx* h, const double* d_x, uint64_t n, void* stream) {
    if (!h) return XSUM_EINVAL;
    if (n == 0) return XSUM_OK;
    if (!d_x || !aligned(d_x, 8)) return XSUM_EINVAL;
    if (n > kMaxCount - h->count) return XSUM_ECAPACITY;
    DeviceGuard g(h->device);
    if (!g.ok) return XSUM_ECUDA;
    if (xs::accumulate(d_x, n, acc_params(h, 0, nullptr, nullptr), grid_of(h), static_cast<cudaStream_t>(stream)) !=
        cudaSuccess)
        return XSUM_ECUDA;
    h->count += n;
    return XSUM_OK;
}

xsum_status xsum_sum(xsum_ctx* h, const double* d_x, uint64_t n, void* d_res, uint64_t* d_canon, void* stream) {
    if (!h || !d_res || !aligned(d_res, 8) || (d_canon && !aligned(d_canon, 8))) return XSUM_EINVAL;
    if (n && (!d_x || !aligned(d_x, 8))) return XSUM_EINVAL;
    if (n > kMaxCount) return XSUM_ECAPACITY;
    DeviceGuard g(h->device);
    if (!g.ok) return XSUM_ECUDA;
    if (xs::accumulate(d_x, n, acc_params(h, 1, static_cast<xsum_result*>(d_res), d_canon), grid_of(h),
                       static_cast<cudaStream_t>(stream)) != cudaSuccess)
        return XSUM_ECUDA;
    h->count = n;
    h->count_pending = false;
    return XSUM_OK;
}

size_t xsum_peer_buffer_bytes(uint32_t world) { return xs::peer_buffer_bytes(world); }

xsum_status xsum_sum_allreduce(xsum_ctx* h, const double* d_x, uint64_t n, void* const* d_bufs, uint32_t rank,
                               uint32_t world, uint64_t epoch, void* d_res, uint64_t* d_canon, void* stream) {
    if (!h || !d_res || !aligned(d_res, 8) || (d_canon && !aligned(d_canon, 8))) return XSUM_EINVAL;
    if (n && (!d_x || !aligned(d_x, 8))) return XSUM_EINVAL;
    if (!d_bufs || !aligned(d_bufs, 8) || world == 0 || rank >= world || epoch == 0) return XSUM_EINVAL;
    if (n > kMaxCount) return XSUM_ECAPACITY;
    DeviceGuard g(h->device);
    if (!g.ok) return XSUM_ECUDA;
    xs::AccParams p = acc_params(h, 1, static_cast<xsum_result*>(d_res), d_canon);
    p.peer.bufs = reinterpret_cast<uint8_t* const*>(d_bufs);
    p.peer.rank = rank;
    p.peer.world = world;
    p.peer.epoch = epoch;
    if (xs::accumulate(d_x, n, p, grid_of(h), static_cast<cudaStream_t>(stream)) != cudaSuccess) return XSUM_ECUDA;
    h->count = n;                                   // host mirror: this rank's shard (the merged
    h->count_pending = false;                       // group total is in the result record)
    return XSUM_OK;
}

xsum_status xsum_peer_selftest(const void* d_states, void* const* d_bufs, uint32_t world, uint64_t epoch, void* d_res,
                               void* d_out, void* stream) {
    if (!d_states || !aligned(d_states, 8) || !d_bufs || !aligned(d_bufs, 8) || !d_res || !aligned(d_res, 8) ||
        !d_out || !aligned(d_out, 8) || world == 0 || world > 64 || epoch == 0)
        return XSUM_EINVAL;
    if (xs::peer_selftest(static_cast<const xsum_state_image*>(d_states), reinterpret_cast<uint8_t* const*>(d_bufs),
                          world, epoch, static_cast<xsum_result*>(d_res), static_cast<xsum_state_image*>(d_out),
                          static_cast<cudaStream_t>(stream)) != cudaSuccess)
        return XSUM_ECUDA;
    return XSUM_OK;
}

xsum_status xsum_accumulate_f32(xsum_ctx* h, const float* d_x, uint64_t n, void* stream) {
    if (!h) return XSUM_EINVAL;
    if (n == 0) return XSUM_OK;
    if (!d_x || !aligned(d_x, 4)) return XSUM_EINVAL;
    if (n > kMaxCount - h->count) return XSUM_ECAPACITY;
    DeviceGuard g(h->device);
    if (!g.ok) return XSUM_ECUDA;
    if (xs::accumulate_f32(d_x, n, acc_params(h, 0, nullptr, nullptr), grid_of(h), static_cast<cudaStream_t>(stream)) !=
        cudaSuccess)
        return XSUM_ECUDA;
    h->count += n;
    return XSUM_OK;
}

xsum_status xsum_sum_f32(xsum_ctx* h, const float* d_x, uint64_t n, void* d_res, uint64_t* d_canon, void* stream) {
    if (!h || !d_res || !aligned(d_res, 8) || (d_canon && !aligned(d_canon, 8))) return XSUM_EINVAL;
    if (n && (!d_x || !aligned(d_x, 4))) return XSUM_EINVAL;
    if (n > kMaxCount) return XSUM_ECAPACITY;
    DeviceGuard g(h->device);
    if (!g.ok) return XSUM_ECUDA;
    if (xs::accumulate_f32(d_x, n, acc_params(h, 1, static_cast<xsum_result*>(d_res), d_canon), grid_of(h),
                           static_cast<cudaStream_t>(stream)) != cudaSuccess)
        return XSUM_ECUDA;
    h->count = n;
    h->count_pending = false;
    return XSUM_OK;
}

xsum_status xsum_accumulate_f16(xsum_ctx* h, const uint16_t* d_x, uint64_t n, void* stream) {
    return accumulate_h16_api(h, d_x, n, 0, stream);
}
xsum_status xsum_accumulate_bf16(xsum_ctx* h, const uint16_t* d_x, uint64_t n, void* stream) {
    return accumulate_h16_api(h, d_x, n, 1, stream);
}
xsum_status xsum_sum_f16(xsum_ctx* h, const uint16_t* d_x, uint64_t n, void* d_res, uint64_t* d_canon, void* stream) {
    return sum_h16_api(h, d_x, n, 0, d_res, d_canon, stream);
}
xsum_status xsum_sum_bf16(xsum_ctx* h, const uint16_t* d_x, uint64_t n, void* d_res, uint64_t* d_canon, void* stream) {
    return sum_h16_api(h, d_x, n, 1, d_res, d_canon, stream);
}

// Host-buffer streaming for any element format (dtype XSUM_DT_*): double-buffered H2D chunks on
// the handle's copy stream, each accumulated on `stream` while the next one is in flight.
static xsum_status accumulate_host_any(xsum_ctx* h, const void* h_x, uint64_t n, int dtype, void* d_stage,
                                       size_t stage_bytes, void* stream) {
    if (!h) return XSUM_EINVAL;
    if (dtype < XSUM_DT_F64 || dtype > XSUM_DT_BF16) return XSUM_EINVAL;
    if (n == 0) return XSUM_OK;
    if (!h_x || !d_stage || !aligned(d_stage, 256) || stage_bytes < (2u << 20)) return XSUM_EINVAL;
    if (n > kMaxCount - h->count) return XSUM_ECAPACITY;
    const uint64_t esz = dtype == XSUM_DT_F64 ? 8 : (dtype == XSUM_DT_F32 ? 4 : 2);
    DeviceGuard g(h->device);
    if (!g.ok) return XSUM_ECUDA;
    if (!h->copy_stream) {
        if (cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking) != cudaSuccess) return XSUM_ECUDA;
        for (int b = 0; b < 2; ++b) {
            if (cudaEventCreateWithFlags(&h->ev_ready[b], cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&h->ev_done[b], cudaEventDisableTiming) != cudaSuccess)
                return XSUM_ECUDA;
        }
        // first use: nothing consumed the staging halves yet
        for (int b = 0; b < 2; ++b)
            if (cudaEventRecord(h->ev_done[b], h->copy_stream) != cudaSuccess) return XSUM_ECUDA;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint64_t half = (stage_bytes / 2) / 256 * 256;
    const uint64_t per = half / esz;
    uint8_t* base = static_cast<uint8_t*>(d_stage);
    const uint8_t* src = static_cast<const uint8_t*>(h_x);
    // order the copies after all prior work on `stream`
    if (cudaEventRecord(h->ev_ready[0], s) != cudaSuccess || cudaStreamWaitEvent(h->copy_stream, h->ev_ready[0], 0) != cudaSuccess)
        return XSUM_ECUDA;
    uint64_t off = 0;
    int b = 0;
    while (off < n) {
        uint64_t cnt = (n - off) < per ? (n - off) : per;
        uint8_t* buf = base + (uint64_t)b * half;
        if (cudaStreamWaitEvent(h->copy_stream, h->ev_done[b], 0) != cudaSuccess ||
            cudaMemcpyAsync(buf, src + off * esz, cnt * esz, cudaMemcpyHostToDevice, h->copy_stream) != cudaSuccess ||
            cudaEventRecord(h->ev_ready[b], h->copy_stream) != cudaSuccess ||
            cudaStreamWaitEvent(s, h->ev_ready[b], 0) != cudaSuccess)
            return XSUM_ECUDA;
        const xs::AccParams p = acc_params(h, 0, nullptr, nullptr);
        cudaError_t e;
        if (dtype == XSUM_DT_F64) e = xs::accumulate(reinterpret_cast<const double*>(buf), cnt, p, grid_of(h), s);
        else if (dtype == XSUM_DT_F32) e = xs::accumulate_f32(reinterpret_cast<const float*>(buf), cnt, p, grid_of(h), s);
        else e = xs::accumulate_h16(reinterpret_cast<const uint16_t*>(buf), cnt, dtype == XSUM_DT_BF16, p, grid_of(h), s);
        if (e != cudaSuccess) return XSUM_ECUDA;
        if (cudaEventRecord(h->ev_done[b], s) != cudaSuccess) return XSUM_ECUDA;
        off += cnt;
        b ^= 1;
    }
    h->count += n;
    return XSUM_OK;
}

xsum_status xsum_accumulate_host(xsum_ctx* h, const double* h_x, uint64_t n, void* d_stage, size_t stage_bytes,
                                 void* stream) {
    return accumulate_host_any(h, h_x, n, XSUM_DT_F64, d_stage, stage_bytes, stream);
}

xsum_status xsum_accumulate_host_ex(xsum_ctx* h, const void* h_x, uint64_t n, int dtype, void* d_stage,
                                    size_t stage_bytes, void* stream) {
    return accumulate_host_any(h, h_x, n, dtype, d_stage, stage_bytes, stream);
}

xsum_status xsum_merge(xsum_ctx* h, const void* d_states, uint32_t count, void* stream) {
    if (!h) return XSUM_EINVAL;
    if (count == 0) return XSUM_OK;
    if (!d_states || !aligned(d_states, 8)) return XSUM_EINVAL;
    DeviceGuard g(h->device);
    if (!g.ok) return XSUM_ECUDA;
    if (xs::merge_states(h->state, d_states, count, 0, nullptr, nullptr, static_cast<cudaStream_t>(stream)) !=
        cudaSuccess)
        return XSUM_ECUDA;
    return note_merge(h, static_cast<cudaStream_t>(stream));
}

xsum_status xsum_to_sparse(xsum_ctx* h, void* d_out, uint32_t* d_nbytes, void* stream) {
    if (!h || !d_out || !aligned(d_out, 8) || !d_nbytes || !aligned(d_nbytes, 4)) return XSUM_EINVAL;
    DeviceGuard g(h->device);
    if (!g.ok) return XSUM_ECUDA;
    if (xs::to_sparse(h->state, d_out, d_nbytes, static_cast<cudaStream_t>(stream)) != cudaSuccess) return XSUM_ECUDA;
    return XSUM_OK;
}

xsum_status xsum_merge_sparse(xsum_ctx* h, const void* d_images, const uint64_t* d_offsets, uint32_t count,
                              void* stream) {
    if (!h) return XSUM_EINVAL;
    if (count == 0) return XSUM_OK;
    if (!d_images || !aligned(d_images, 8) || !d_offsets || !aligned(d_offsets, 8)) return XSUM_EINVAL;
    DeviceGuard g(h->device);
    if (!g.ok) return XSUM_ECUDA;
    if (xs::merge_sparse(h->state, d_images, d_offsets, count, static_cast<cudaStream_t>(stream)) != cudaSuccess)
        return XSUM_ECUDA;
    return note_merge(h, static_cast<cudaStream_t>(stream));
}

xsum_status xsum_merge_round(xsum_ctx* h, const void* d_states, uint32_t count, void* d_res, uint64_t* d_canon,
                             void* stream) {
    if (!h || !d_res || !aligned(d_res, 8) || (d_canon && !aligned(d_canon, 8))) return XSUM_EINVAL;
    if (count && (!d_states || !aligned(d_states, 8))) return XSUM_EINVAL;
    DeviceGuard g(h->device);
    if (!g.ok) return XSUM_ECUDA;
    if (xs::merge_states(h->state, d_states, count, 1, static_cast<xsum_result*>(d_res), d_canon,
                         static_cast<cudaStream_t>(stream)) != cudaSuccess)
        return XSUM_ECUDA;
    return note_merge(h, static_cast<cudaStream_t>(stream));
}

xsum_status xsum_finalize_round(xsum_ctx* h, void* d_res, uint64_t* d_canon, void* stream) {
    if (!h || !d_res || !aligned(d_res, 8) || (d_canon && !aligned(d_canon, 8))) return XSUM_EINVAL;
    DeviceGuard g(h->device);
    if (!g.ok) return XSUM_ECUDA;
    if (xs::finalize(h->state, static_cast<xsum_result*>(d_res), d_canon, static_cast<cudaStream_t>(stream)) !=
        cudaSuccess)
        return XSUM_ECUDA;
    return XSUM_OK;
}

xsum_status xsum_destroy(xsum_ctx* h) {
    if (!h) return XSUM_EINVAL;
    {
        DeviceGuard g(h->device);
        if (h->copy_stream) {
            cudaStreamSynchronize(h->copy_stream);
            for (int b = 0; b < 2; ++b) {
                cudaEventDestroy(h->ev_ready[b]);
                cudaEventDestroy(h->ev_done[b]);
            }
            cudaStreamDestroy(h->copy_stream);
        }
        if (h->count_pinned) {
            cudaEventSynchronize(h->ev_count);
            cudaEventDestroy(h->ev_count);
            cudaFreeHost(h->count_pinned);
        }
    }
    delete h;
    return XSUM_OK;
}

uint64_t xsum_count(const xsum_ctx* ch) {
    if (!ch) return 0;
    xsum_ctx* h = const_cast<xsum_ctx*>(ch);
    if (h->count_pending) {             // resolve the merged count (waits for the merge's copy)
        DeviceGuard g(h->device);
        if (!g.ok || cudaEventSynchronize(h->ev_count) != cudaSuccess) return UINT64_MAX;
        const uint64_t base = *h->count_pinned;
        h->count = (base > kMaxCount - h->count) ? kMaxCount : base + h->count;
        h->count_pending = false;
    }
    return h->count;
}

xsum_status xsum_set_grid_limit(xsum_ctx* h, uint32_t max_blocks) {
    if (!h) return XSUM_EINVAL;
    h->grid_limit = max_blocks;
    return XSUM_OK;
}

xsum_status xsum_sum_segments(const double* d_x, uint64_t nseg, uint64_t seg_len, double* d_out, uint64_t* d_canon,
                              uint32_t* d_flags, void* stream) {
    if (nseg == 0) return XSUM_OK;
    if (!d_out || !aligned(d_out, 8) || (d_canon && !aligned(d_canon, 8)) || (d_flags && !aligned(d_flags, 4)))
        return XSUM_EINVAL;
    if (seg_len && (!d_x || !aligned(d_x, 8))) return XSUM_EINVAL;
    if (seg_len && nseg > kMaxCount / seg_len) return XSUM_EINVAL;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return XSUM_ECUDA;
    if (xs::sum_segments(d_x, nseg, seg_len, nullptr, xs::SegOut{d_out, nullptr, d_canon, d_flags}, sms_of(dev),
                         static_cast<cudaStream_t>(stream)) != cudaSuccess)
        return XSUM_ECUDA;
    return XSUM_OK;
}

xsum_status xsum_sum_segments_csr(const double* d_x, const uint64_t* d_offsets, uint64_t nseg, double* d_out,
                                  uint64_t* d_canon, uint32_t* d_flags, void* stream) {
    if (nseg == 0) return XSUM_OK;
    if (!d_offsets || !aligned(d_offsets, 8) || !d_out || !aligned(d_out, 8) || (d_canon && !aligned(d_canon, 8)) ||
        (d_flags && !aligned(d_flags, 4)))
        return XSUM_EINVAL;
    if (!d_x || !aligned(d_x, 8)) return XSUM_EINVAL;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return XSUM_ECUDA;
    if (xs::sum_segments(d_x, nseg, 0, d_offsets, xs::SegOut{d_out, nullptr, d_canon, d_flags}, sms_of(dev),
                         static_cast<cudaStream_t>(stream)) != cudaSuccess)
        return XSUM_ECUDA;
    return XSUM_OK;
}

xsum_status xsum_sum_segments_ex(const void* d_x, int dtype, uint64_t nseg, uint64_t seg_len,
                                 const uint64_t* d_offsets, double* d_out, float* d_out32, uint64_t* d_canon,
                                 uint32_t* d_flags, void* stream) {
    return xsum_sum_segments_ws(d_x, dtype, nseg, seg_len, d_offsets, d_out, d_out32, d_canon, d_flags, nullptr,
                                stream);
}

xsum_status xsum_sum_segments_ws(const void* d_x, int dtype, uint64_t nseg, uint64_t seg_len,
                                 const uint64_t* d_offsets, double* d_out, float* d_out32, uint64_t* d_canon,
                                 uint32_t* d_flags, void* d_ticket, void* stream) {
    if (d_ticket && !aligned(d_ticket, 8)) return XSUM_EINVAL;
    if (dtype < XSUM_DT_F64 || dtype > XSUM_DT_BF16) return XSUM_EINVAL;
    if (nseg == 0) return XSUM_OK;
    if (!d_out && !d_out32 && !d_canon && !d_flags) return XSUM_EINVAL;
    if ((d_out && !aligned(d_out, 8)) || (d_out32 && !aligned(d_out32, 4)) || (d_canon && !aligned(d_canon, 8)) ||
        (d_flags && !aligned(d_flags, 4)) || (d_offsets && !aligned(d_offsets, 8)))
        return XSUM_EINVAL;
    const uintptr_t esz = dtype == XSUM_DT_F64 ? 8 : (dtype == XSUM_DT_F32 ? 4 : 2);
    if ((d_offsets || seg_len) && (!d_x || !aligned(d_x, esz))) return XSUM_EINVAL;
    if (!d_offsets && seg_len && nseg > kMaxCount / seg_len) return XSUM_EINVAL;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return XSUM_ECUDA;
    const xs::SegOut o{d_out, d_out32, d_canon, d_flags};
    cudaError_t e;
    if (dtype == XSUM_DT_F64)
        e = xs::sum_segments(static_cast<const double*>(d_x), nseg, d_offsets ? 0 : seg_len, d_offsets, o, sms_of(dev),
                             static_cast<cudaStream_t>(stream), static_cast<unsigned long long*>(d_ticket));
    else
        e = xs::sum_segments_small(d_x, dtype, nseg, d_offsets ? 0 : seg_len, d_offsets, o, sms_of(dev),
                                   static_cast<cudaStream_t>(stream), static_cast<unsigned long long*>(d_ticket));
    return e == cudaSuccess ? XSUM_OK : XSUM_ECUDA;
}

xsum_status xsum_sum_segments_csr_lanes(const void* d_x, int dtype, uint64_t nseg, const uint64_t* d_offsets,
                                        double* d_out, float* d_out32, uint64_t* d_canon, uint32_t* d_flags,
                                        void* d_ticket, void* stream) {
    if (dtype < XSUM_DT_F64 || dtype > XSUM_DT_BF16) return XSUM_EINVAL;
    if (nseg == 0) return XSUM_OK;
    if (!d_out && !d_out32 && !d_canon && !d_flags) return XSUM_EINVAL;
    const uintptr_t esz = dtype == XSUM_DT_F64 ? 8 : (dtype == XSUM_DT_F32 ? 4 : 2);
    if (!d_offsets || !aligned(d_offsets, 8) || !d_x || !aligned(d_x, esz) || (d_out && !aligned(d_out, 8)) ||
        (d_out32 && !aligned(d_out32, 4)) || (d_canon && !aligned(d_canon, 8)) || (d_flags && !aligned(d_flags, 4)) ||
        (d_ticket && !aligned(d_ticket, 8)))
        return XSUM_EINVAL;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return XSUM_ECUDA;
    const xs::SegOut o{d_out, d_out32, d_canon, d_flags};
    return xs::sum_segments_lanes_csr(d_x, dtype, nseg, d_offsets, o, static_cast<unsigned long long*>(d_ticket),
                                      sms_of(dev), static_cast<cudaStream_t>(stream)) == cudaSuccess ? XSUM_OK
                                                                                                     : XSUM_ECUDA;
}

size_t xsum_condsens_work_bytes(uint64_t n) { return xs::condsens_work_bytes(n); }

xsum_status xsum_sum_condsens(const double* d_x, uint64_t n, int rule, void* d_work, size_t work_bytes, void* d_res,
                              void* d_info, uint64_t* d_canon, void* stream) {
    if (rule != 1 && rule != 2) return XSUM_EINVAL;
    if (!d_res || !aligned(d_res, 8) || !d_info || !aligned(d_info, 8) || (d_canon && !aligned(d_canon, 8)))
        return XSUM_EINVAL;
    if (!d_work || !aligned(d_work, 256) || work_bytes < xs::condsens_work_bytes(n)) return XSUM_EINVAL;
    if (n && (!d_x || !aligned(d_x, 8))) return XSUM_EINVAL;
    if (n > kMaxCount) return XSUM_EINVAL;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return XSUM_ECUDA;
    return xs::condsens_sum(d_x, n, rule, d_work, work_bytes, static_cast<xsum_result*>(d_res),
                            static_cast<xsum_condsens_info*>(d_info), d_canon, sms_of(dev),
                            static_cast<cudaStream_t>(stream)) == cudaSuccess ? XSUM_OK : XSUM_ECUDA;
}

size_t xsum_sum_strided_work_bytes(uint64_t outer, uint64_t len, uint64_t inner, int device) {
    if (inner <= 1) return 0;
    return xs::strided_work_bytes(outer, len, inner, sms_of(device));
}

xsum_status xsum_sum_strided(const void* d_x, int dtype, uint64_t outer, uint64_t len, uint64_t inner,
                             double* d_out64, float* d_out32, uint32_t* d_flags, void* d_work, size_t work_bytes,
                             void* stream) {
    if (dtype < XSUM_DT_F64 || dtype > XSUM_DT_BF16) return XSUM_EINVAL;
    if (!d_out64 && !d_out32) return XSUM_EINVAL;
    if ((d_out64 && !aligned(d_out64, 8)) || (d_out32 && !aligned(d_out32, 4)) || (d_flags && !aligned(d_flags, 4)) ||
        (d_work && !aligned(d_work, 8)))
        return XSUM_EINVAL;
    if (outer == 0 || inner == 0) return XSUM_OK;
    if (outer > kMaxCount / inner || (len && outer * inner > kMaxCount / len)) return XSUM_EINVAL;
    const uintptr_t esz = dtype == XSUM_DT_F64 ? 8 : (dtype == XSUM_DT_F32 ? 4 : 2);
    if (len && (!d_x || !aligned(d_x, esz))) return XSUM_EINVAL;
    if (inner == 1)                                 // contiguous fibres: the segment kernels
        return xsum_sum_segments_ex(d_x, dtype, outer, len, nullptr, d_out64, d_out32, nullptr, d_flags, stream);
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return XSUM_ECUDA;
    const xs::StrOut o{d_out64, d_out32, d_flags};
    return xs::sum_strided(d_x, dtype, outer, len, inner, o, d_work, work_bytes, sms_of(dev),
                           static_cast<cudaStream_t>(stream)) == cudaSuccess ? XSUM_OK : XSUM_ECUDA;
}

}  // extern "C"
