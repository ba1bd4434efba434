// K4 (merge tree of superaccumulators) and K5 (finalize: canonicalize + round).
//
// Merge: the MapReduce post-process (§6.1; Spark driver merge
// PAPER.md:1186-1189) as a Lemma-1 pairwise tree: states are added
// digit-parallel with signed carries C in {-1,0,1} that move at most one digit.
// Finalize: steps 6-7 of the PRAM algorithm, see finalize_warp.
#include <cuda_runtime.h>
#include <cstddef>

#include "grid_tail.cuh"
#include "xsum_device.cuh"
#include "xsum_kernels.h"

namespace xs {

__global__ void k_init_state(xsum_state_image* st) {
    int t = threadIdx.x;
    if (t < D) st->digit[t] = 0;
    uint8_t* pad = st->pad;
    if (t < (int)sizeof(st->pad)) pad[t] = 0;
    if (t == 0) {
        st->magic = XSUM_MAGIC;
        st->version = (uint16_t)XSUM_VERSION;
        st->w = (uint8_t)W;
        st->ndigits = (uint8_t)D;
        st->flags = 0;
        st->reserved = 0;
        st->count = 0;
    }
}

// A state image is accepted (DenseImages::load_from) iff its header matches and its digits are regularized
// (|Y_j| <= R-1 below the top digit; top digit bounded by the value).

constexpr int MERGE_WARPS = 16;

// Leaf loaders of the merge tree: one warp reads image s into digit-parallel registers
// (a0 = digit lane, a1 = digit lane+32). Returns false (image rejected) on a bad header or
// digits that are not regularized.
struct DenseImages {
    const xsum_state_image* ims;
    // k_merge's leaf pipeline (as for sparse images): image s + 16's header and digits are in flight
    // while image s is validated and folded
    struct Hdr {
        uint64_t off, w0, w1, w2;      // off: the image index; w0: magic | version | w | ndigits,
        int64_t d0, d1;                // w1: flags | reserved, w2: count; digits lane and lane + 32
    };
    __device__ __forceinline__ uint64_t off_of(uint32_t s, uint32_t /*count*/) const { return s; }
    __device__ __forceinline__ Hdr hdr_of(uint64_t s, bool valid, int lane) const {
        Hdr h{s, 0, 0, 0, 0, 0};
        if (valid) {
            const xsum_state_image* im = ims + s;
            const uint64_t* p = reinterpret_cast<const uint64_t*>(im);
            h.w0 = p[0];
            h.w1 = p[1];
            h.w2 = p[2];
            h.d0 = im->digit[lane];
            h.d1 = (lane + 32 < D) ? im->digit[lane + 32] : 0;
        }
        return h;
    }
    __device__ __forceinline__ bool load_from(const Hdr& h, int lane, int64_t* /*scratch*/, int64_t& d0, int64_t& d1,
                                              uint64_t& cnt, uint32_t& fl) const {
        d0 = h.d0;
        d1 = h.d1;
        cnt = h.w2;
        fl = (uint32_t)h.w1;
        const bool hdr = (uint32_t)h.w0 == XSUM_MAGIC && ((h.w0 >> 32) & 0xFFFFu) == XSUM_VERSION &&
                         ((h.w0 >> 48) & 0xFFu) == (uint64_t)W && (h.w0 >> 56) == (uint64_t)D;
        const bool ok0 = d0 >= -(R - 1) && d0 <= R - 1;
        const bool ok1 = (lane + 32 < D - 1) ? (d1 >= -(R - 1) && d1 <= R - 1)
                                             : ((lane + 32 == D - 1) ? (d1 >= -XSUM_TOP_DIGIT_MAX && d1 <= XSUM_TOP_DIGIT_MAX)
                                                                     : true);
        return hdr && cnt <= COUNT_MAX && __all_sync(FULL, ok0 && ok1);     
    }
};
static_assert(offsetof(xsum_state_image, ndigits) == 7 && offsetof(xsum_state_image, flags) == 8 &&
              offsetof(xsum_state_image, count) == 16 && offsetof(xsum_state_image, digit) == 24,
              "DenseImages::Hdr word layout");

// Sparse images (the paper's sparse superaccumulator, PAPER.md:682-696:
// only the active indices are kept): a 24-byte header and nnz records (digit << 6) | index in
// ascending index order (include/xsum.h). Image s starts at base + offs[s].
struct SparseImages {
    const uint8_t* base;
    const uint64_t* offs;
    // The three dependent loads of an image (offset -> header -> records) are software-pipelined by
    // k_merge: offsets two images ahead, headers one ahead (ncu r02f: 1024 images in 117 us, stalls
    // on long_scoreboard 14 per issued instruction, with the chain serialised per image).
    struct Hdr {
        uint64_t off, w0, w1, w2;      // w0: magic | version | w | nnz, w1: flags | reserved, w2: count
    };
    __device__ __forceinline__ uint64_t off_of(uint32_t s, uint32_t count) const { return s < count ? offs[s] : 0; }
    __device__ __forceinline__ Hdr hdr_of(uint64_t off, bool valid, int /*lane*/) const {
        Hdr h{off, 0, 0, 0};
        if (valid && !(off & 7)) {
            const uint64_t* p = reinterpret_cast<const uint64_t*>(base + off);
            h.w0 = p[0];
            h.w1 = p[1];
            h.w2 = p[2];
        }
        return h;
    }
    __device__ __forceinline__ bool load_from(const Hdr& h, int lane, int64_t* scratch, int64_t& d0, int64_t& d1,
                                              uint64_t& cnt, uint32_t& fl) const {
        d0 = d1 = 0;
        cnt = 0;
        fl = 0;
        if (h.off & 7) return false;                                   // warp-uniform
        const uint32_t magic = (uint32_t)h.w0, version = (uint32_t)(h.w0 >> 32) & 0xFFFFu;
        const uint32_t w = (uint32_t)(h.w0 >> 48) & 0xFFu, nnz = (uint32_t)(h.w0 >> 56);
        if (magic != XSUM_SPARSE_MAGIC || version != XSUM_VERSION || w != W || nnz > (uint32_t)D) return false;
        const uint64_t* rec = reinterpret_cast<const uint64_t*>(base + h.off + sizeof(xsum_sparse_header));
        scratch[lane] = 0;
        scratch[lane + 32] = 0;
        __syncwarp();
        bool ok = true;
        int prev_last = -1;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const uint32_t r = (uint32_t)lane + 32u * hh;
            const bool has = r < nnz;
            const uint64_t v = has ? rec[r] : 0;
            const int idx = has ? (int)(v & 63u) : 64;
            const int64_t dg = (int64_t)v >> 6;
            int prev = __shfl_up_sync(FULL, idx, 1);
            if (lane == 0) prev = prev_last;
            prev_last = __shfl_sync(FULL, idx, 31);
            if (has) {
                const int64_t lim = idx < D - 1 ? R - 1 : XSUM_TOP_DIGIT_MAX;
                ok = ok && idx < D && idx > prev && dg != 0 && dg >= -lim && dg <= lim;
                if (idx < D) scratch[idx] = dg;
            }
        }
        __syncwarp();
        d0 = scratch[lane];
        d1 = (lane + 32 < D) ? scratch[lane + 32] : 0;
        cnt = h.w2;
        fl = (uint32_t)h.w1;
        return __all_sync(FULL, ok) && cnt <= COUNT_MAX;
    }
};
static_assert(sizeof(xsum_sparse_header) == 24 && offsetof(xsum_sparse_header, nnz) == 7 &&
              offsetof(xsum_sparse_header, flags) == 8 && offsetof(xsum_sparse_header, count) == 16,
              "SparseImages::Hdr word layout");

template <class Src>
__global__ void __launch_bounds__(MERGE_WARPS * 32)
k_merge(xsum_state_image* st, Src src, uint32_t count, int overwrite, xsum_result* res, uint64_t* canon) {
    __shared__ int64_t acc[MERGE_WARPS][64];
    __shared__ int64_t scr[MERGE_WARPS][64];
    __shared__ uint64_t cnts[MERGE_WARPS];
    __shared__ uint32_t fls[MERGE_WARPS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t a0 = 0, a1 = 0;
    uint64_t cnt = 0;
    uint32_t fl = 0;
    // leaves: each warp folds images warp, warp+16, ... (Lemma-1 adds)
    auto fold = [&](bool ok, int64_t d0, int64_t d1, uint64_t c, uint32_t f) {
        if (ok) {
            lemma1_add(a0, a1, d0, d1, lane);
            cnt = count_add(cnt, c, fl);
            fl |= f & (XSUM_F_NAN | XSUM_F_PINF | XSUM_F_NINF | XSUM_F_MISMATCH | XSUM_F_PEER_TIMEOUT |
                       XSUM_F_CAPACITY);
        } else {
            fl |= XSUM_F_MISMATCH;
        }
    };
    uint64_t off1 = src.off_of(warp + MERGE_WARPS, count);
    typename Src::Hdr h = src.hdr_of(src.off_of(warp, count), warp < count, lane);
    for (uint32_t s = warp; s < count; s += MERGE_WARPS) {
        const uint64_t off2 = src.off_of(s + 2 * MERGE_WARPS, count);          // two images ahead
        const typename Src::Hdr hn = src.hdr_of(off1, s + MERGE_WARPS < count, lane);  // one ahead
        int64_t d0, d1;
        uint64_t c;
        uint32_t f;
        const bool ok = src.load_from(h, lane, scr[warp], d0, d1, c, f);
        fold(ok, d0, d1, c, f);
        h = hn;
        off1 = off2;
    }
    acc[warp][lane] = a0;
    acc[warp][lane + 32] = a1;
    if (lane == 0) { cnts[warp] = cnt; fls[warp] = fl; }
    __syncthreads();
    // pairwise tree over the warp results (depth log2(16))
    for (int stride = MERGE_WARPS / 2; stride >= 1; stride >>= 1) {
        if (warp < stride) {
            int64_t b0 = acc[warp + stride][lane], b1 = acc[warp + stride][lane + 32];
            lemma1_add(a0, a1, b0, b1, lane);
            acc[warp][lane] = a0;
            acc[warp][lane + 32] = a1;
            if (lane == 0) {
                uint32_t f2 = fls[warp] | fls[warp + stride];
                cnts[warp] = count_add(cnts[warp], cnts[warp + stride], f2);
                fls[warp] = f2;
            }
        }
        __syncthreads();
    }
    if (warp == 0) {
        uint64_t cnt_all = cnts[0];
        uint32_t fl_all = fls[0];
        if (!overwrite) {
            int64_t s0 = st->digit[lane], s1 = (lane + 32 < D) ? st->digit[lane + 32] : 0;
            lemma1_add(a0, a1, s0, s1, lane);
            fl_all |= st->flags;
            cnt_all = count_add(cnt_all, st->count, fl_all);
        }
        st->digit[lane] = a0;
        if (lane + 32 < D) st->digit[lane + 32] = a1;
        if (lane < (int)(sizeof(st->pad))) st->pad[lane] = 0;
        if (lane == 0) {
            st->magic = XSUM_MAGIC;
            st->version = (uint16_t)XSUM_VERSION;
            st->w = (uint8_t)W;
            st->ndigits = (uint8_t)D;
            st->reserved = 0;
            st->count = cnt_all;
            st->flags = fl_all;
        }
        if (res) {                                // fused post-process rounding
            __shared__ int64_t su[64];
            xsum_result r = finalize_warp(a0, a1, fl_all, cnt_all, canon, su, lane);
            if (lane == 0) *res = r;
        }
    }
}

__global__ void k_finalize(const xsum_state_image* st, xsum_result* res, uint64_t* canon) {
    __shared__ int64_t su[64];
    const int lane = threadIdx.x & 31;
    int64_t a0 = st->digit[lane];
    int64_t a1 = (lane + 32 < D) ? st->digit[lane + 32] : 0;
    xsum_result r = finalize_warp(a0, a1, st->flags, st->count, canon, su, lane);
    if (lane == 0) *res = r;
}

cudaError_t init_state(xsum_state_image* st, cudaStream_t s) {
    k_init_state<<<1, 64, 0, s>>>(st);
    note_launch();
    return cudaGetLastError();
}

cudaError_t merge_states(xsum_state_image* st, const void* states, uint32_t count, int overwrite, xsum_result* res,
                         uint64_t* canon, cudaStream_t s) {
    k_merge<<<1, MERGE_WARPS * 32, 0, s>>>(st, DenseImages{static_cast<const xsum_state_image*>(states)}, count,
                                           overwrite, res, canon);
    note_launch();
    return cudaGetLastError();
}

cudaError_t merge_sparse(xsum_state_image* st, const void* images, const uint64_t* offsets, uint32_t count,
                         cudaStream_t s) {
    k_merge<<<1, MERGE_WARPS * 32, 0, s>>>(st, SparseImages{static_cast<const uint8_t*>(images), offsets}, count, 0,
                                           nullptr, nullptr);
    note_launch();
    return cudaGetLastError();
}

// Encode the (regularized) state as a sparse image: one record per non-zero digit, ascending.
__global__ void k_to_sparse(const xsum_state_image* st, uint8_t* out, uint32_t* nbytes) {
    const int lane = threadIdx.x & 31;
    const int64_t a0 = st->digit[lane];
    const int64_t a1 = (lane + 32 < D) ? st->digit[lane + 32] : 0;
    const uint64_t nz = (uint64_t)__ballot_sync(FULL, a0 != 0) | ((uint64_t)__ballot_sync(FULL, a1 != 0) << 32);
    const uint32_t nnz = __popcll(nz);
    uint64_t* rec = reinterpret_cast<uint64_t*>(out + sizeof(xsum_sparse_header));
    if (a0 != 0) rec[__popcll(nz & ((1ull << lane) - 1))] = ((uint64_t)a0 << 6) | (uint64_t)lane;
    if (a1 != 0) rec[__popcll(nz & ((1ull << (lane + 32)) - 1))] = ((uint64_t)a1 << 6) | (uint64_t)(lane + 32);
    if (lane == 0) {
        xsum_sparse_header* hd = reinterpret_cast<xsum_sparse_header*>(out);
        hd->magic = XSUM_SPARSE_MAGIC;
        hd->version = (uint16_t)XSUM_VERSION;
        hd->w = (uint8_t)W;
        hd->nnz = (uint8_t)nnz;
        hd->flags = st->flags;
        hd->reserved = 0;
        hd->count = st->count;
        *nbytes = (uint32_t)(sizeof(xsum_sparse_header) + 8 * nnz);
    }
}

cudaError_t to_sparse(const xsum_state_image* st, void* out, uint32_t* nbytes, cudaStream_t s) {
    k_to_sparse<<<1, 32, 0, s>>>(st, static_cast<uint8_t*>(out), nbytes);
    note_launch();
    return cudaGetLastError();
}

// One block per virtual rank: the exchange of the fused multi-GPU step on one device.
__global__ void k_peer_selftest(const xsum_state_image* states, uint8_t* const* bufs, uint32_t world, uint64_t epoch,
                                xsum_result* res, xsum_state_image* out) {
    __shared__ int64_t su[64];
    const int lane = threadIdx.x & 31;
    const uint32_t r = blockIdx.x;
    const xsum_state_image* in = states + r;
    int64_t b0 = in->digit[lane], b1 = (lane + 32 < D) ? in->digit[lane + 32] : 0;
    uint32_t fl = in->flags;
    uint64_t cnt = in->count;
    PeerParams pp;
    pp.bufs = bufs;
    pp.rank = r;
    pp.world = world;
    pp.epoch = epoch;
    peer_exchange_merge(b0, b1, fl, cnt, pp, lane);
    xsum_state_image* o = out + r;
    o->digit[lane] = b0;
    if (lane + 32 < D) o->digit[lane + 32] = b1;
    if (lane < (int)sizeof(o->pad)) o->pad[lane] = 0;
    if (lane == 0) {
        o->magic = XSUM_MAGIC;
        o->version = (uint16_t)XSUM_VERSION;
        o->w = (uint8_t)W;
        o->ndigits = (uint8_t)D;
        o->reserved = 0;
        o->flags = fl;
        o->count = cnt;
    }
    xsum_result rr = finalize_warp(b0, b1, fl, cnt, nullptr, su, lane);
    if (lane == 0) res[r] = rr;
}

cudaError_t peer_selftest(const xsum_state_image* states, uint8_t* const* bufs, uint32_t world, uint64_t epoch,
                          xsum_result* res, xsum_state_image* out, cudaStream_t s) {
    void* args[] = {(void*)&states, (void*)&bufs, (void*)&world, (void*)&epoch, (void*)&res, (void*)&out};
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_peer_selftest, dim3(world), dim3(32), args, 0, s);
    note_launch();
    return e;
}

cudaError_t finalize(const xsum_state_image* st, xsum_result* res, uint64_t* canon, cudaStream_t s) {
    k_finalize<<<1, 32, 0, s>>>(st, res, canon);
    note_launch();
    return cudaGetLastError();
}

}  // namespace xs
