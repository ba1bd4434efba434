// Grid level of the merge tree (§3 step 5 bottom-up; MapReduce
// post-process PAPER.md:1158-1163): every block publishes its regularized superaccumulator
// to the scratch table, and the last block to arrive merges the table and the handle state
// and, for a fused one-shot sum, rounds. Shared by the accumulate kernels.
#pragma once

#include "xsum_device.cuh"
#include "xsum_kernels.h"

namespace xs {

__device__ __forceinline__ int64_t warp_sum64(int64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

// Call with all threads of the block. On entry warp 0 holds the block's regularized digits
// (a0 = digit lane, a1 = digit lane+32) and `bflags` the block's flags; other warps' a0/a1
// are ignored. `red` is >= D int64 of shared scratch, `su` 64 int64, `sh_flags`/`sh_last`
// shared words. `n` is the launch's summand count (added to the state's count).
template <int WARPS>
__device__ __forceinline__ void grid_tail(int64_t a0, int64_t a1, uint32_t bflags, uint64_t n, const AccParams& p,
                                          int64_t* red, int64_t* su, uint32_t* sh_flags, int* sh_last, int warp,
                                          int lane) {
    const uint64_t G = gridDim.x;
    if (warp == 0) {
        p.partial[(size_t)lane * XS_MAXB + blockIdx.x] = a0;
        if (lane + 32 < D) p.partial[(size_t)(lane + 32) * XS_MAXB + blockIdx.x] = a1;
        if (lane == 0) p.pflags[blockIdx.x] = bflags;
        __syncwarp();
        if (lane == 0) {
            // release: this block's partial (ordered before by the warp barrier) is visible to
            // the block that sees the final count; acquire: the last block sees all of them
            uint32_t old;
            asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(p.counter) : "memory");
            *sh_last = (old == (uint32_t)(G - 1));
        }
    }
    __syncthreads();
    if (!*sh_last) return;
    __threadfence();

    // The last block merges the G block partials (digit-major, coalesced) and the handle
    // state; G <= XS_MAXB so the raw sum stays below 2^62 before regularizing. Warp w sums
    // digits w, w+WARPS, ...; a lane issues all its loads of one round (4 partials of each of
    // its digits) before using any: one L2 round trip per 128 blocks instead of one per 32.
    constexpr int JPW = (D + WARPS - 1) / WARPS;
    int64_t st0 = 0, st1 = 0;
    if (warp == 0 && !p.overwrite) {                     // state digits, fetched alongside
        st0 = __ldcg(&p.state->digit[lane]);
        st1 = (lane + 32 < D) ? __ldcg(&p.state->digit[lane + 32]) : 0;
    }
    int64_t acc[JPW];
#pragma unroll
    for (int jj = 0; jj < JPW; ++jj) acc[jj] = 0;
    for (uint64_t b0 = lane; b0 < G; b0 += 128) {
        int64_t v[JPW][4];
#pragma unroll
        for (int jj = 0; jj < JPW; ++jj)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int j = warp + jj * WARPS;
                const uint64_t b = b0 + 32 * u;
                v[jj][u] = (j < D && b < G) ? __ldcg(&p.partial[(size_t)j * XS_MAXB + b]) : 0;
            }
#pragma unroll
        for (int jj = 0; jj < JPW; ++jj) acc[jj] += (v[jj][0] + v[jj][1]) + (v[jj][2] + v[jj][3]);
    }
#pragma unroll
    for (int jj = 0; jj < JPW; ++jj) {
        const int j = warp + jj * WARPS;
        const int64_t s = warp_sum64(acc[jj]);
        if (j < D && lane == 0) red[j] = s;
    }
    if (warp == 1 % WARPS) {
        uint32_t f = 0;
        for (uint64_t b = lane; b < G; b += 32) f |= __ldcg(&p.pflags[b]);
        f = __reduce_or_sync(FULL, f);
        if (lane == 0) *sh_flags = f;
    }
    __syncthreads();
    if (warp == 0) {
        int64_t b0 = red[lane] + st0, b1 = (lane + 32 < D) ? red[lane + 32] + st1 : 0;
        uint32_t fl = *sh_flags;
        uint64_t cnt = n;
        if (!p.overwrite) {
            fl |= p.state->flags;
            cnt += p.state->count;
        }
        regularize_warp(b0, b1, lane);
        p.state->digit[lane] = b0;
        if (lane + 32 < D) p.state->digit[lane + 32] = b1;
        if (lane == 0) {
            p.state->flags = fl;
            p.state->count = cnt;
            *p.counter = 0;                      // ready for the next launch (stream order)
        }
        if (p.res) {
            xsum_result r = finalize_warp(b0, b1, fl, cnt, p.canon, su, lane);
            if (lane == 0) *p.res = r;
        }
    }
}

}  // namespace xs
