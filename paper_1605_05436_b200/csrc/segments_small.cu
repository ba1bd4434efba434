// K9: segmented exact sums of binary32 / binary16 / bfloat16 elements (SURVEY.md §8(f) f1 x f2:
// reproducible reductions of the formats tensors are usually stored in).
//
// One warp per segment (the paper's per-partition combine), lanes striding
// over the segment with 16-byte loads. Each element of the paper's t-bit / l-bit format
// is M 2^k in units of its least subnormal, i.e. M at bit k + OFF of the
// 2^-1074 window (binary32 OFF = 925, binary16 1050, bfloat16 941); it is split into the two
// 52-bit digit chunks of PAPER.md:744-750 and added to the lane's column with carries deferred
// (regularized every FLUSH_ELEMS adds). NaN/Inf patterns are flagged, not
// added (reading R10). At the segment's end the 32 columns are combined and finalize_warp
// canonicalizes and rounds (binary64 and binary32).
#include <cuda_runtime.h>

#include "xsum_device.cuh"
#include "xsum_kernels.h"

namespace xs {

template <int T_, int L_, int OFF_, int EB_>
struct SFmt {
    static constexpr int t = T_, l = L_, off = OFF_, eb = EB_;
    static constexpr int per_vec = 16 / EB_;
};
using SF32 = SFmt<23, 8, 925, 4>;
using SF16 = SFmt<10, 5, 1050, 2>;
using SBF16 = SFmt<7, 8, 941, 2>;

// Element bits b (the low 8*eb bits): chunks of sign * M * 2^(k + off); spec = 1 for NaN/Inf.
template <class F>
__device__ __forceinline__ Chunks sdecode(uint32_t b, uint32_t one) {
    constexpr uint32_t SBIT = F::t + F::l;
    constexpr uint32_t EM = (1u << F::l) - 1u;
    Chunks c;
    const uint32_t h = b & ((1u << SBIT) - 1u);
    const uint32_t e = h >> F::t;
    const uint32_t ep = max(e, 1u);
    const uint32_t M = h - ((ep - 1u) << F::t);                  // m + [e != 0] 2^t
    const uint32_t K = mad_u32(ep, one, (uint32_t)F::off - 1u);  // k + off
    const uint32_t i = mulhi_u32(K, K52);                        // K / 52
    const uint32_t o = K - 52u * i;
    const int64_t sM = ((b >> SBIT) & 1u) ? -(int64_t)M : (int64_t)M;
    c.c0 = (int64_t)(((uint64_t)sM << o) & MASK);
    c.c1 = sM >> (52u - o);
    c.i = i;
    c.spec = (e == EM);
    return c;
}

template <class F>
__device__ __forceinline__ uint32_t sspecial_flags(uint32_t b) {
    constexpr uint32_t SBIT = F::t + F::l;
    constexpr uint32_t EM = (1u << F::l) - 1u;
    if (((b >> F::t) & EM) != EM) return 0;
    if (b & ((1u << F::t) - 1u)) return XSUM_F_NAN;
    return ((b >> SBIT) & 1u) ? XSUM_F_NINF : XSUM_F_PINF;
}

template <class F>
__device__ __forceinline__ void sadd(int64_t* col, uint32_t b, uint32_t& flags, uint32_t one) {
    const Chunks c = sdecode<F>(b, one);
    if (c.spec) { flags |= sspecial_flags<F>(b); return; }
    column_add(col, c, one);
}

// the elements of a 16-byte vector
template <class F>
__device__ __forceinline__ void sadd_vec(int64_t* col, const uint4& v, uint32_t& flags, uint32_t one) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (F::eb == 4) {
            sadd<F>(col, w[q], flags, one);
        } else {
            sadd<F>(col, w[q] & 0xFFFFu, flags, one);
            sadd<F>(col, w[q] >> 16, flags, one);
        }
    }
}

template <class F>
__device__ __forceinline__ uint32_t sload_one(const uint8_t* p) {
    if (F::eb == 4) return __ldg(reinterpret_cast<const uint32_t*>(p));
    return __ldg(reinterpret_cast<const uint16_t*>(p));
}

constexpr int SSEG_WARPS = 8;
constexpr size_t SSEG_SMEM = (size_t)SSEG_WARPS * D * 32 * sizeof(int64_t);

template <class F>
__global__ void __launch_bounds__(SSEG_WARPS * 32, 2)
k_segments_small(const uint8_t* __restrict__ x, uint64_t nseg, uint64_t seg_len, const uint64_t* __restrict__ offsets,
                 SegOut o, uint32_t one) {
    extern __shared__ __align__(16) int64_t win[];
    __shared__ int64_t su[SSEG_WARPS][64];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t* col = win + warp * (D * 32) + lane;
    const int64_t* wb = win + warp * (D * 32);
    const uint64_t nw = (uint64_t)gridDim.x * SSEG_WARPS;
    constexpr int PV = F::per_vec;

    constexpr int SU = 4;                                   // vectors per lane per tile
    constexpr uint32_t WIN_TILES = (FLUSH_ELEMS - 2 - SU * PV) / (SU * PV);   // + leftovers + head/tail
    struct Seg {
        const uint8_t* xs;
        uint64_t len, head, nvec, tail, nit;
        const uint4* body;
    };
    auto open_seg = [&](uint64_t sj) {
        Seg g;
        const uint64_t beg = offsets ? offsets[sj] : sj * seg_len;
        g.len = offsets ? offsets[sj + 1] - beg : seg_len;
        g.xs = x + beg * F::eb;
        g.head = ((16 - ((uintptr_t)g.xs & 15)) & 15) / F::eb;
        if (g.head > g.len) g.head = g.len;
        g.nvec = (g.len - g.head) / PV;
        g.tail = g.len - g.head - g.nvec * PV;
        g.body = reinterpret_cast<const uint4*>(g.xs + g.head * F::eb);
        g.nit = g.nvec / (32 * SU);
        return g;
    };
    uint64_t s = (uint64_t)blockIdx.x * SSEG_WARPS + warp;
    if (s >= nseg) return;                                  // warp-uniform
#pragma unroll
    for (int j = 0; j < D; ++j) col[j * 32] = 0;
    Seg g = open_seg(s);
    uint4 cur[SU], alt[SU];
    if (g.nit) {
#pragma unroll
        for (int u = 0; u < SU; ++u) cur[u] = ldg_stream(g.body + u * 32 + lane);
    }
    while (true) {
        uint32_t flags = 0, since = 0;
        const uint64_t nit = g.nit, nvec = g.nvec;
        const uint4* body = g.body;
        // head / tail: one element per lane (head < PV <= 8, tail < PV)
        if ((uint64_t)lane < g.head) sadd<F>(col, sload_one<F>(g.xs + lane * F::eb), flags, one);
        if (lane >= 8 && (uint64_t)(lane - 8) < g.tail)
            sadd<F>(col, sload_one<F>(g.xs + (g.head + nvec * PV + (lane - 8)) * F::eb), flags, one);
        // full tiles: two register buffers alternate (tile it+1 loads while tile it is added)
        auto process = [&](const uint4 (&bf)[SU]) {
#pragma unroll
            for (int u = 0; u < SU; ++u) sadd_vec<F>(col, bf[u], flags, one);
            if (++since == WIN_TILES) { regularize_column(col); since = 0; }
        };
        for (uint64_t it = 0; it < nit; it += 2) {
            if (it + 1 < nit) {
#pragma unroll
                for (int u = 0; u < SU; ++u) alt[u] = ldg_stream(body + (it + 1) * (32 * SU) + u * 32 + lane);
            }
            process(cur);
            if (it + 1 >= nit) break;
            if (it + 2 < nit) {
#pragma unroll
                for (int u = 0; u < SU; ++u) cur[u] = ldg_stream(body + (it + 2) * (32 * SU) + u * 32 + lane);
            }
            process(alt);
        }
        // leftover vectors (< one tile), loaded together before use
        uint4 lv[SU];
#pragma unroll
        for (int u = 0; u < SU; ++u) {
            const uint64_t v = nit * (32 * SU) + u * 32 + lane;
            if (v < nvec) lv[u] = ldg_stream(body + v);
        }
#pragma unroll
        for (int u = 0; u < SU; ++u)
            if (nit * (32 * SU) + u * 32 + lane < nvec) sadd_vec<F>(col, lv[u], flags, one);
        // prefetch the next segment, then close this one
        const uint64_t sn = s + nw;
        const bool more = sn < nseg;
        const uint64_t len = g.len;
        if (more) {
            g = open_seg(sn);
            if (g.nit) {
#pragma unroll
                for (int u = 0; u < SU; ++u) cur[u] = ldg_stream(g.body + u * 32 + lane);
            }
        }
        __syncwarp();
        int64_t a0, a1;
        combine_raw_columns(wb, a0, a1, lane);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < D; ++j) col[j * 32] = 0;
        flags = __reduce_or_sync(FULL, flags);
        const xsum_result r =
            finalize_warp_inl(a0, a1, flags, len, o.canon ? o.canon + s * XSUM_CANON_LIMBS : nullptr, su[warp], lane);
        if (lane == 0) o.write(s, r);
        __syncwarp();
        if (!more) break;
        s = sn;
    }
}

template <class F>
static cudaError_t launch_small(const void* x, uint64_t nseg, uint64_t seg_len, const uint64_t* offsets,
                                const SegOut& o, int num_sms, cudaStream_t s) {
    static unsigned long long smem_set = 0;
    if (cudaError_t e = ensure_smem(k_segments_small<F>, SSEG_SMEM, smem_set)) return e;
    const uint64_t want = (nseg + SSEG_WARPS - 1) / SSEG_WARPS;
    const uint64_t cap = (uint64_t)num_sms * 2;
    const unsigned g = (unsigned)(want < cap ? (want ? want : 1) : cap);
    k_segments_small<F><<<g, SSEG_WARPS * 32, SSEG_SMEM, s>>>(static_cast<const uint8_t*>(x), nseg, seg_len, offsets, o,
                                                               1u);
    note_launch();
    return cudaGetLastError();
}

cudaError_t sum_segments_small(const void* x, int dtype, uint64_t nseg, uint64_t seg_len, const uint64_t* offsets,
                               const SegOut& o, int num_sms, cudaStream_t s) {
    switch (dtype) {
        case XSUM_DT_F32: return launch_small<SF32>(x, nseg, seg_len, offsets, o, num_sms, s);
        case XSUM_DT_F16: return launch_small<SF16>(x, nseg, seg_len, offsets, o, num_sms, s);
        case XSUM_DT_BF16: return launch_small<SBF16>(x, nseg, seg_len, offsets, o, num_sms, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace xs
