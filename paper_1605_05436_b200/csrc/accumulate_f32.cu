// K8: exact sums of binary32 inputs with exponent-group bins.
//
// A binary32 is M 2^k in units of 2^-149 (t = 23, l = 8; M < 2^24,
// k = max(e,1) - 1). Splitting every summand into two 52-bit digit chunks (the binary64 path)
// costs two 64-bit read-modify-writes of shared memory per summand; with only 24 significand
// bits one is enough: each lane keeps unsigned 64-bit bins, one per (sign, group of 32
// consecutive exponents), and adds M 2^(ep mod 32) (ep = max(e,1)) into bin (ep >> 5, sign) -
// an integer component at an exponent that is a multiple of a fixed width,
// carries deferred, no sign handling in the hot loop. Every FLUSH adds
// (M 2^o < 2^55, 511 adds < 2^64) a lane empties its bins into its digit column (each bin at a
// fixed bit position: the split into <= 3 digits uses constant shifts), and every REG_FLUSHES
// flushes regularizes the column.
// binary32 values live in digits 17..24 of the 52-bit window (bit positions 924..1148+63), so
// the per-lane column holds only the COLS digits from COL0 on (the top one takes the carries
// and is never split); the warp combine moves them to their digit positions for the binary64
// block reduction and grid tail (grid_tail.cuh).
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
#define XS_F32B_NB 3
#endif
constexpr int F32B_NB = XS_F32B_NB;        // rotating register buffers
constexpr int F32B_NG = 8;                 // groups: ep = max(e,1) in [1, 255] -> ep >> 5 in [0, 7]
constexpr int F32B_NBIN = 2 * F32B_NG;     // bin 2 g + sign
constexpr int F32B_FLUSH = 511;            // 511 * (2^24 - 1) 2^31 < 2^64
constexpr int F32B_REG_FLUSHES = 128;      // <= 10 chunks per digit per flush: 2^51 + 1280 * 2^52 < 2^63
constexpr int F32B_BASE = 925;             // window bit position of k = 0 (2^-149 = 2^925 * 2^-1074)
constexpr uint32_t F32B_SPEC_EP = 255;     // exponent field of NaN/Inf
constexpr int F32B_COL0 = 17;              // first digit of the per-lane column
constexpr int F32B_COLS = 12;              // digits 17..28: bins reach digit 24; carries above

static_assert(F32B_FLUSH * ((((1ull << 24) - 1) << 31) >> 8) < (1ull << 56), "bin window too long");
static_assert((16 + 1) * (((1ull << 24) - 1) << 31) < (1ull << 63), "leftovers (after a flush) overflow a bin");
__host__ __device__ constexpr int f32b_pos(int g) { return F32B_BASE - 1 + 32 * g; }   // bin g's bit position
static_assert(f32b_pos(0) / 52 >= F32B_COL0 && f32b_pos(F32B_NG - 1) / 52 + 2 < F32B_COL0 + F32B_COLS - 2,
              "column window does not cover the bins and their carries");

// One summand: bits b. ep = max(e,1); M = h + 2^23 - ep 2^23 = m + [e!=0] 2^23; bin (ep >> 5, s)
// gets M 2^(ep mod 32) = |x| 2^149 / 2^(32 g - 1). `bins` = this lane's bin column (bin b at word
// b*32); byte offset of bin (g, s) = 512 g + 256 s = 16 (ep - o) + 256 s.
__device__ __forceinline__ void f32b_add(uint64_t* bins, uint32_t b, uint32_t& spec, uint32_t one) {
    const uint32_t h = b & 0x7FFFFFFFu;
    const uint32_t ep = max(h >> 23, 1u);
    const uint32_t M = mad_u32(ep, 0u - (1u << 23), mad_u32(h, one, 1u << 23));
    const uint32_t o = ep & 31u;
    uint32_t vhi;                                               // high word of M 2^o
    asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(vhi) : "r"(M), "r"(0u), "r"(o));
    const uint64_t v = ((uint64_t)vhi << 32) | (M << o);
    spec = max(spec, ep);
    const uint32_t off = mad_u32(mad_u32(o, 0xFFFFFFFFu, ep), 16u, (b >> 31) << 8);   // bytes
    XS_ASSERT(off / 256 < (uint32_t)F32B_NBIN);
    uint64_t* p = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(bins) + off);
    *p += v;
}

__device__ __forceinline__ uint32_t f32b_special_flags(uint32_t b) {
    if (((b >> 23) & 0xFFu) != 0xFFu) return 0;
    if (b & 0x7FFFFFu) return XSUM_F_NAN;
    return (b >> 31) ? XSUM_F_NINF : XSUM_F_PINF;
}

// Empty the bins into the digit column (row r = digit COL0 + r): bin (g, s) is worth
// (-1)^s V 2^pos(g); V 2^o (o = pos mod 52) splits into c0 + c1 2^52 + c2 2^104, all >= 0.
__device__ __forceinline__ void f32b_flush(uint64_t* bins, int64_t* col) {
#pragma unroll
    for (int b = 0; b < F32B_NBIN; ++b) {
        const int P = f32b_pos(b >> 1), i = P / W - F32B_COL0, o = P % W;
        const uint64_t V = bins[b * 32];
        bins[b * 32] = 0;
        const int64_t c0 = (int64_t)((V << o) & MASK);
        const int64_t c1 = (int64_t)((V >> (W - o)) & MASK);
        const int64_t c2 = (int64_t)(2 * W - o < 64 ? V >> (2 * W - o) : 0);
        XS_ASSERT(i >= 0 && i + 2 < F32B_COLS - 1);
        XS_ASSERT(col[i * 32] > -0x7F00000000000000ll && col[i * 32] < 0x7F00000000000000ll);
        if (b & 1) {
            col[i * 32] -= c0;
            col[(i + 1) * 32] -= c1;
            col[(i + 2) * 32] -= c2;
        } else {
            col[i * 32] += c0;
            col[(i + 1) * 32] += c1;
            col[(i + 2) * 32] += c2;
        }
    }
}

// Regularize the narrow column; its top digit only takes carries.
__device__ __forceinline__ void f32b_regularize(int64_t* col) {
    int64_t cin = 0;
#pragma unroll
    for (int j = 0; j < F32B_COLS - 1; ++j) {
        const int64_t y = col[j * 32];
        const int64_t c = balanced_carry(y);
        col[j * 32] = y - (c << W) + cin;
        cin = c;
    }
    col[(F32B_COLS - 1) * 32] += cin;
}

// Rare path: this lane summed NaN/Inf patterns as finite values (ep = 255) in tiles [t0, t1];
// re-read them, set the flags and cancel them (the sign-flipped pattern lands in the other
// sign's bin of the same group: net zero), then flush the cancellation into the column.
__device__ __noinline__ void f32b_rescan(uint64_t* bins, int64_t* col, const uint4* body, uint64_t t0, uint64_t t1,
                                         uint64_t G, uint64_t TV, int tid, uint32_t& flags, uint32_t one) {
    uint32_t dummy = 0;
    for (uint64_t tt = t0; tt <= t1; tt += G) {
        for (int u = 0; u < F32B_U; ++u) {
            uint4 v = ld_stream(body + tt * TV + (uint64_t)u * (F32B_WARPS * 32) + tid);
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

__device__ __forceinline__ void f32b_add_checked(uint64_t* bins, uint32_t b, uint32_t& flags, uint32_t one) {
    const uint32_t f = f32b_special_flags(b);
    if (f) { flags |= f; return; }
    uint32_t dummy = 0;
    f32b_add(bins, b, dummy, one);
}

__global__ void __launch_bounds__(F32B_WARPS * 32, 1)
k_accumulate_f32b(const float* x, uint64_t n, AccParams p) {
    constexpr int T = F32B_WARPS * 32;
    constexpr int PV = 4;
    constexpr int FLUSH_TILES = F32B_FLUSH / (PV * F32B_U);           // 31 tiles
    constexpr int GROUPS_PER_WINDOW = FLUSH_TILES / F32B_NB;           // 10 groups of 3
    static_assert(GROUPS_PER_WINDOW >= 1, "window shorter than one buffer group");
    extern __shared__ __align__(16) int64_t win[];                     // [WARPS][COLS][32] columns, then bins
    __shared__ int64_t wsum[F32B_WARPS][D];
    __shared__ int64_t su[64];
    __shared__ uint32_t blk_flags;
    __shared__ int is_last;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    pdl_release_dependents();    // the next launch may take SMs as this grid's blocks finish
    int64_t* col = win + warp * (F32B_COLS * 32) + lane;
    uint64_t* bins = reinterpret_cast<uint64_t*>(win + F32B_WARPS * F32B_COLS * 32) + warp * (F32B_NBIN * 32) + lane;
#pragma unroll
    for (int j = 0; j < F32B_COLS; ++j) col[j * 32] = 0;
#pragma unroll
    for (int g = 0; g < F32B_NBIN; ++g) bins[g * 32] = 0;
    if (tid == 0) blk_flags = 0;
    uint32_t flags = 0;
    pdl_wait_predecessor();      // inputs are read only after the preceding launch completed
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
            for (int u = 0; u < F32B_U; ++u) buf[u] = ld_stream(body + tt * TV + (uint64_t)u * T + tid);
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
            if (spec == F32B_SPEC_EP) {              // the rescan flushes once more
                f32b_rescan(bins, col, body, wstart, tlast, G, TV, tid, flags, one);
                ++flushes;
            }
            if (++flushes >= F32B_REG_FLUSHES) { f32b_regularize(col); flushes = 0; }
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
                const uint4 q = ld_stream(body + v);
                f32b_add_checked(bins, q.x, flags, one);
                f32b_add_checked(bins, q.y, flags, one);
                f32b_add_checked(bins, q.z, flags, one);
                f32b_add_checked(bins, q.w, flags, one);
            }
        }
        const uint64_t tail = nbody - nvec * PV;
        if ((uint64_t)tid < head) f32b_add_checked(bins, __float_as_uint(ld_coherent(x + tid)), flags, one);
        if (tid >= 4 && (uint64_t)(tid - 4) < tail)
            f32b_add_checked(bins, __float_as_uint(ld_coherent(x + head + nvec * PV + (tid - 4))), flags, one);
        f32b_flush(bins, col);
    }
    __syncwarp();

    // warp: lane r < COLS sums row r (digit COL0 + r) over the 32 lanes as hi/lo 32-bit halves
    // (raw digits |Y| < 2^63), splits off balanced carries, and the carries move one row up;
    // the rows then move to their digit positions (digit j in lane j).
    {
        const int64_t* wb = win + warp * (F32B_COLS * 32);
        int64_t hs = 0, ls = 0;
        if (lane < F32B_COLS) {
#pragma unroll 8
            for (int c = 0; c < 32; ++c) {
                const int64_t v = wb[lane * 32 + ((lane + c) & 31)];
                hs += v >> 32;
                ls += (int64_t)(uint32_t)v;
            }
        }
        int64_t cr = 0, rr = (int64_t)((uint64_t)hs << 32) + ls;       // top row: not split
        if (lane < F32B_COLS - 1) {
            cr = (hs + ((ls + (1ll << 51)) >> 32)) >> 20;
            rr = (int64_t)((uint64_t)(hs - (cr << 20)) << 32) + ls;
        }
        int64_t cin = __shfl_up_sync(FULL, cr, 1);
        if (lane == 0) cin = 0;
        const int64_t row = lane < F32B_COLS ? rr + cin : 0;
        const int64_t d = __shfl_sync(FULL, row, (lane - F32B_COL0) & 31);
        const int64_t s0 = (lane >= F32B_COL0 && lane < F32B_COL0 + F32B_COLS) ? d : 0;
        wsum[warp][lane] = s0;
        if (lane + 32 < D) wsum[warp][lane + 32] = 0;
        const uint32_t f = __reduce_or_sync(FULL, flags);
        if (lane == 0 && f) atomicOr(&blk_flags, f);
    }
    __syncthreads();
    int64_t a0 = 0, a1 = 0;
    if (warp == 0) {
#pragma unroll
        for (int w = 0; w < F32B_WARPS; ++w) a0 += wsum[w][lane];
        regularize_warp(a0, a1, lane);
    }
    grid_tail<F32B_WARPS>(a0, a1, blk_flags, n, p, wsum[0], su, &blk_flags, &is_last, warp, lane);
}

cudaError_t accumulate_f32(const float* x, uint64_t n, const AccParams& p, int num_sms, cudaStream_t s) {
    constexpr size_t SMEM = (size_t)F32B_WARPS * 32 * (F32B_COLS + F32B_NBIN) * sizeof(int64_t);
    static unsigned long long smem_set = 0;
    if (cudaError_t e = ensure_smem(k_accumulate_f32b, SMEM, smem_set)) return e;
    uint64_t head = ((16 - ((uintptr_t)x & 15)) & 15) / 4;
    if (head > n) head = n;
    const uint64_t ntiles = ((n - head) / 4) / ((uint64_t)F32B_WARPS * 32 * F32B_U);
    uint64_t g = ntiles < (uint64_t)num_sms ? ntiles : (uint64_t)num_sms;
    if (g < 1) g = 1;
    if (g > XS_MAXB) g = XS_MAXB;
    cudaError_t e = launch_pdl(n * 4 < PDL_MAX_BYTES, k_accumulate_f32b, (unsigned)g, F32B_WARPS * 32, SMEM, s, x, n, p);
    note_launch();
    return e;
}

}  // namespace xs
