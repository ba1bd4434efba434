// K8: exact sums of binary32 inputs with exponent-group bins.
//
// A binary32 is M 2^k in units of 2^-149 (t = 23, l = 8; M < 2^24,
// k = max(e,1) - 1). Splitting every summand into two 52-bit digit chunks (the binary64 path)
// costs two 64-bit read-modify-writes of shared memory per summand; with only 24 significand
// bits one is enough: each lane keeps signed int64 bins, one per group of 32 consecutive
// exponents, and adds +-M 2^(ep mod 32) (ep = max(e,1)) into bin ep >> 5 - an integer component
// at an exponent that is a multiple of a fixed width, carries deferred
// (PAPER.md:669-673). Every FLUSH adds (|M 2^o| < 2^55, 255 adds < 2^63) a lane empties its bins
// into its 52-bit digit column (each bin at a fixed bit position, so the split into <= 3
// digits uses constant shifts), and every REG_FLUSHES flushes regularizes the column
// (PAPER.md:559-576). The columns then go through the binary64 path's combine and grid tail.
// NaN/Inf patterns (ep = 255) are summed as if finite; a per-lane max of ep sends a lane that
// saw one to rescan its window, set the flags and cancel them exactly (reading R10).
#include <cuda_runtime.h>

#include "grid_tail.cuh"
#include "xsum_device.cuh"
#include "xsum_kernels.h"

namespace xs {

constexpr int F32B_WARPS = 16;
constexpr int F32B_U = 4;                 // 16-B vectors (4 summands) per thread per tile
#ifndef XS_F32B_NB
#define XS_F32B_NB 3   // c32 2^29: NB=3 1129, 4 1119, 5 1071 G/s
#endif
constexpr int F32B_NB = XS_F32B_NB;        // rotating register buffers
constexpr int F32B_NG = 8;                 // groups: ep = max(e,1) in [1, 255] -> ep >> 5 in [0, 7]
constexpr int F32B_NBIN = F32B_NG;
constexpr int F32B_FLUSH = 255;            // 255 * 2^55 < 2^63
constexpr int F32B_REG_FLUSHES = 256;      // <= 4 chunks per digit per flush: 2^51 + 1024 * 2^52 < 2^63
constexpr int F32B_BASE = 925;             // window bit position of k = 0 (2^-149 = 2^925 * 2^-1074)
constexpr uint32_t F32B_SPEC_EP = 255;      // exponent field of NaN/Inf

static_assert(F32B_FLUSH * (((1ull << 24) - 1) << 31) < (1ull << 63), "bin window too long");
static_assert((16 + 1) * (((1ull << 24) - 1) << 31) < (1ull << 63), "leftovers (after a flush) overflow a bin");
__host__ __device__ constexpr int f32b_pos(int g) { return F32B_BASE - 1 + 32 * g; }   // bin g's bit position

// One summand: bits b. ep = max(e,1); M = h + 2^23 - ep 2^23 = m + [e!=0] 2^23; bin ep >> 5 gets
// sign(x) M 2^(ep mod 32) = x 2^149 / 2^(32 g - 1). NaN/Inf (ep = 255) share bin 7 with finite
// values: the running max of ep sends the lane to the rare path (cancel + flag) at the window
// close. Ops are split between the ALU pipe and the FMA pipe (IMAD / IMAD.HI with the opaque
// `one`): the kernel is issue/ALU bound. `bins` = this lane's bin column (bin g at word g*32).
__device__ __forceinline__ void f32b_add(int64_t* bins, uint32_t b, uint32_t& spec, uint32_t one) {
    const uint32_t h = b & 0x7FFFFFFFu;
    const uint32_t ep = max(h >> 23, 1u);
    const uint32_t M = mad_u32(ep, 0u - (1u << 23), mad_u32(h, one, 1u << 23));
    const int32_t sgn = (int32_t)mad_u32((uint32_t)mulhi_s32((int32_t)b, 2), 2u, 1u);   // +-1
    const int32_t sM = (int32_t)mad_u32(M, (uint32_t)sgn, 0u);                           // +-M
    const uint32_t o = ep & 31u;
    uint32_t vhi;                                     // high word of sM 2^o: funnel of (sM >> 31 : sM)
    asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(vhi) : "r"((uint32_t)sM), "r"((uint32_t)mulhi_s32(sM, 2)), "r"(o));
    const int64_t v = (int64_t)(((uint64_t)vhi << 32) | ((uint32_t)sM << o));
    spec = max(spec, ep);
    int64_t* p = bins + mad_u32(mad_u32(o, 0xFFFFFFFFu, ep), one, 0u);   // (ep - o) = 32 g: word 32 g
    XS_ASSERT((ep >> 5) < (uint32_t)F32B_NBIN);
    *p += v;
}

__device__ __forceinline__ uint32_t f32b_special_flags(uint32_t b) {
    if (((b >> 23) & 0xFFu) != 0xFFu) return 0;
    if (b & 0x7FFFFFu) return XSUM_F_NAN;
    return (b >> 31) ? XSUM_F_NINF : XSUM_F_PINF;
}

// Empty the finite bins into the digit column: bin g is worth V 2^pos(g); V 2^o (o = pos mod 52)
// splits into c0 + c1 2^52 + c2 2^104 with c0, c1 in [0, 2^52) and c2 signed.
__device__ __forceinline__ void f32b_flush(int64_t* bins, int64_t* col) {
#pragma unroll
    for (int g = 0; g < F32B_NG; ++g) {
        const int P = f32b_pos(g), i = P / W, o = P % W;
        const int64_t V = bins[g * 32];
        bins[g * 32] = 0;
        const int64_t c0 = (int64_t)(((uint64_t)V << o) & MASK);
        const int64_t c1 = (V >> (W - o)) & (int64_t)MASK;
        const int64_t c2 = V >> (2 * W - o < 63 ? 2 * W - o : 63);
        XS_ASSERT(i + 2 < D - 1);
        XS_ASSERT(col[i * 32] > -0x7FC0000000000000ll && col[i * 32] < 0x7FC0000000000000ll);
        XS_ASSERT(col[(i + 1) * 32] > -0x7FC0000000000000ll && col[(i + 1) * 32] < 0x7FC0000000000000ll);
        XS_ASSERT(col[(i + 2) * 32] > -0x7FC0000000000000ll && col[(i + 2) * 32] < 0x7FC0000000000000ll);
        col[i * 32] += c0;
        col[(i + 1) * 32] += c1;
        col[(i + 2) * 32] += c2;
    }
}

// Rare path: this lane summed NaN/Inf patterns as finite values (ep = 255) in tiles [t0, t1];
// re-read them, set the flags and cancel them (the sign-flipped pattern's bin contribution),
// then flush the cancellation into the column.
__device__ __noinline__ void f32b_rescan(int64_t* bins, int64_t* col, const uint4* body, uint64_t t0, uint64_t t1,
                                         uint64_t G, uint64_t TV, int tid, uint32_t& flags, uint32_t one) {
    uint32_t dummy = 0;
    for (uint64_t tt = t0; tt <= t1; tt += G) {
        for (int u = 0; u < F32B_U; ++u) {
            uint4 v = ldg_stream(body + tt * TV + (uint64_t)u * (F32B_WARPS * 32) + tid);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
            for (int i = 0; i < 4; ++i) {
                const uint32_t f = f32b_special_flags(w[i]);
                if (f) {
                    flags |= f;
                    f32b_add(bins, w[i] ^ 0x80000000u, dummy, one);
                }
            }
        }
    }
    f32b_flush(bins, col);
}

__device__ __forceinline__ void f32b_add_checked(int64_t* bins, uint32_t b, uint32_t& flags, uint32_t one) {
    const uint32_t f = f32b_special_flags(b);
    if (f) { flags |= f; return; }
    uint32_t dummy = 0;
    f32b_add(bins, b, dummy, one);
}

__global__ void __launch_bounds__(F32B_WARPS * 32, 1)
k_accumulate_f32b(const float* __restrict__ x, uint64_t n, AccParams p) {
    constexpr int T = F32B_WARPS * 32;
    constexpr int PV = 4;
    constexpr int FLUSH_TILES = F32B_FLUSH / (PV * F32B_U);           // 15 tiles
    constexpr int GROUPS_PER_WINDOW = FLUSH_TILES / F32B_NB;           // 3 groups of 5
    static_assert(GROUPS_PER_WINDOW >= 1, "window shorter than one buffer group");
    extern __shared__ __align__(16) int64_t win[];                     // [WARPS][D][32] columns, then bins
    __shared__ int64_t wsum[F32B_WARPS][D];
    __shared__ int64_t su[64];
    __shared__ uint32_t blk_flags;
    __shared__ int is_last;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    pdl_release_dependents();    // the next launch may take SMs as this grid's blocks finish
    int64_t* col = win + warp * (D * 32) + lane;
    int64_t* bins = win + F32B_WARPS * D * 32 + warp * (F32B_NBIN * 32) + lane;
#pragma unroll
    for (int j = 0; j < D; ++j) col[j * 32] = 0;
#pragma unroll
    for (int g = 0; g < F32B_NBIN; ++g) bins[g * 32] = 0;
    if (tid == 0) blk_flags = 0;
    uint32_t flags = 0;
    const uint32_t one = p.one;

    uint64_t head = ((16 - ((uintptr_t)x & 15)) & 15) / 4;
    if (head > n) head = n;
    const uint64_t nbody = n - head;
    const uint64_t nvec = nbody / PV;
    const uint4* body = reinterpret_cast<const uint4*>(x + head);
    const uint64_t TV = (uint64_t)T * F32B_U;
    const uint64_t ntiles = nvec / TV;
    const uint64_t G = gridDim.x;

    uint32_t spec = 0;
    uint64_t wstart = blockIdx.x, tlast = 0;
    bool any_tile = false;
    int flushes = 0;
    auto load_tile = [&](uint4 (&buf)[F32B_U], uint64_t tt) {
        if (tt < ntiles) {
#pragma unroll
            for (int u = 0; u < F32B_U; ++u) buf[u] = ldg_stream(body + tt * TV + (uint64_t)u * T + tid);
        }
    };
    uint4 buf[F32B_NB][F32B_U];
    uint64_t t = blockIdx.x;
#pragma unroll
    for (int b = 0; b < F32B_NB; ++b) load_tile(buf[b], t + (uint64_t)b * G);
    bool more = t < ntiles;
    int groups = 0;
    while (more) {
#pragma unroll
        for (int b = 0; b < F32B_NB; ++b) {
            if (more) {
#pragma unroll
                for (int u = 0; u < F32B_U; ++u) {
                    f32b_add(bins, buf[b][u].x, spec, one);
                    f32b_add(bins, buf[b][u].y, spec, one);
                    f32b_add(bins, buf[b][u].z, spec, one);
                    f32b_add(bins, buf[b][u].w, spec, one);
                }
                any_tile = true;
                tlast = t;
                load_tile(buf[b], t + (uint64_t)F32B_NB * G);
                t += G;
                more = t < ntiles;
            }
        }
        if (++groups == GROUPS_PER_WINDOW) {
            f32b_flush(bins, col);
            if (++flushes == F32B_REG_FLUSHES) { regularize_column_inl(col); flushes = 0; }
            if (spec == F32B_SPEC_EP) f32b_rescan(bins, col, body, wstart, tlast, G, TV, tid, flags, one);
            spec = 0;
            groups = 0;
            wstart = t;
            any_tile = false;
        }
    }
    f32b_flush(bins, col);
    if (spec == F32B_SPEC_EP && any_tile) f32b_rescan(bins, col, body, wstart, tlast, G, TV, tid, flags, one);

    // leftovers (< one tile), the unaligned head and the tail: checked adds by the block that
    // would own the next tile (<= 17 summands per thread), then one more flush
    if (blockIdx.x == ntiles % G) {
        const uint64_t v0 = ntiles * TV;
#pragma unroll
        for (int u = 0; u < F32B_U; ++u) {
            const uint64_t v = v0 + (uint64_t)u * T + tid;
            if (v < nvec) {
                const uint4 q = ldg_stream(body + v);
                f32b_add_checked(bins, q.x, flags, one);
                f32b_add_checked(bins, q.y, flags, one);
                f32b_add_checked(bins, q.z, flags, one);
                f32b_add_checked(bins, q.w, flags, one);
            }
        }
        const uint64_t tail = nbody - nvec * PV;
        if ((uint64_t)tid < head) f32b_add_checked(bins, __float_as_uint(__ldg(x + tid)), flags, one);
        if (tid >= 4 && (uint64_t)(tid - 4) < tail)
            f32b_add_checked(bins, __float_as_uint(__ldg(x + head + nvec * PV + (tid - 4))), flags, one);
        f32b_flush(bins, col);
    }
    __syncwarp();

    // warp: sum the 32 raw lane columns; block: the warps; grid: grid_tail.cuh
    {
        int64_t s0, s1;
        combine_raw_columns(win + warp * (D * 32), s0, s1, lane);
        wsum[warp][lane] = s0;
        if (lane + 32 < D) wsum[warp][lane + 32] = s1;
        const uint32_t f = __reduce_or_sync(FULL, flags);
        if (lane == 0 && f) atomicOr(&blk_flags, f);
    }
    __syncthreads();
    int64_t a0 = 0, a1 = 0;
    if (warp == 0) {
#pragma unroll
        for (int w = 0; w < F32B_WARPS; ++w) {
            a0 += wsum[w][lane];
            if (lane + 32 < D) a1 += wsum[w][lane + 32];
        }
        regularize_warp(a0, a1, lane);
    }
    grid_tail<F32B_WARPS>(a0, a1, blk_flags, n, p, wsum[0], su, &blk_flags, &is_last, warp, lane);
}

cudaError_t accumulate_f32(const float* x, uint64_t n, const AccParams& p, int num_sms, cudaStream_t s) {
    constexpr size_t SMEM = (size_t)F32B_WARPS * 32 * (D + F32B_NBIN) * sizeof(int64_t);
    static unsigned long long smem_set = 0;
    if (cudaError_t e = ensure_smem(k_accumulate_f32b, SMEM, smem_set)) return e;
    uint64_t head = ((16 - ((uintptr_t)x & 15)) & 15) / 4;
    if (head > n) head = n;
    const uint64_t ntiles = ((n - head) / 4) / ((uint64_t)F32B_WARPS * 32 * F32B_U);
    uint64_t g = ntiles < (uint64_t)num_sms ? ntiles : (uint64_t)num_sms;
    if (g < 1) g = 1;
    if (g > XS_MAXB) g = XS_MAXB;
    cudaError_t e = launch_pdl(k_accumulate_f32b, (unsigned)g, F32B_WARPS * 32, SMEM, s, x, n, p);
    note_launch();
    return e;
}

}  // namespace xs
