// K6: segmented exact sums (BASELINE.json config 5) and CSR variable-length segments.
//
// One warp reduces one segment with the same lane-column hot loop as K2, then combines
// its 32 columns, regularizes and rounds without
// leaving the warp - the paper's per-partition "combine" with a
// warp as the partition's worker. Warps loop over segments (persistent grid).
#include <cuda_runtime.h>

#include "xsum_device.cuh"
#include "xsum_kernels.h"

namespace xs {

constexpr int SEG_WARPS = 8;
constexpr int SEG_U = 4;
constexpr int SEG_FLUSH_ITERS = FLUSH_ELEMS / (2 * SEG_U);
constexpr size_t SEG_SMEM = (size_t)SEG_WARPS * D * 32 * sizeof(int64_t);

__device__ __forceinline__ void seg_rescan(int64_t* col, const uint4* body, uint64_t it0, uint64_t it1, int lane,
                                           uint32_t& flags, uint32_t one) {
    for (uint64_t it = it0; it <= it1; ++it) {
#pragma unroll
        for (int u = 0; u < SEG_U; ++u) {
            uint4 v = ldg_stream(body + it * (32 * SEG_U) + u * 32 + lane);
            column_fix_special(col, v.x, v.y, flags, one);
            column_fix_special(col, v.z, v.w, flags, one);
        }
    }
}

__global__ void __launch_bounds__(SEG_WARPS * 32, 2)
k_segments(const double* __restrict__ x, uint64_t nseg, uint64_t seg_len, const uint64_t* __restrict__ offsets,
           double* __restrict__ out, uint64_t* __restrict__ canon, uint32_t* __restrict__ oflags, uint32_t one,
           uint32_t mone) {
    extern __shared__ __align__(16) int64_t win[];
    __shared__ int64_t su[SEG_WARPS][64];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t* col = win + warp * (D * 32) + lane;
    const uint64_t nw = (uint64_t)gridDim.x * SEG_WARPS;

    for (uint64_t s = (uint64_t)blockIdx.x * SEG_WARPS + warp; s < nseg; s += nw) {
        const uint64_t beg = offsets ? offsets[s] : s * seg_len;
        const uint64_t len = offsets ? offsets[s + 1] - beg : seg_len;
        const double* xs = x + beg;
#pragma unroll
        for (int j = 0; j < D; ++j) col[j * 32] = 0;
        uint32_t flags = 0, nspec = 0;

        const uint64_t head = (len && ((uintptr_t)xs & 15)) ? 1 : 0;
        const uint64_t nbody = len - head;
        const uint64_t nvec = nbody >> 1;
        const uint4* body = reinterpret_cast<const uint4*>(xs + head);
        const uint64_t nit = nvec / (32 * SEG_U);

        uint64_t wstart = 0;
        int since = 0;
        uint4 cur[SEG_U];
        if (nit) {
#pragma unroll
            for (int u = 0; u < SEG_U; ++u) cur[u] = ldg_stream(body + u * 32 + lane);
        }
        for (uint64_t it = 0; it < nit; ++it) {
            uint4 nxt[SEG_U];
            if (it + 1 < nit) {
#pragma unroll
                for (int u = 0; u < SEG_U; ++u) nxt[u] = ldg_stream(body + (it + 1) * (32 * SEG_U) + u * 32 + lane);
            }
#pragma unroll
            for (int u = 0; u < SEG_U; ++u) {
                Chunks a = decompose(cur[u].x, cur[u].y, one, mone);
                nspec = spec_fold(nspec, a);
                column_add(col, a, one);
                Chunks b = decompose(cur[u].z, cur[u].w, one, mone);
                nspec = spec_fold(nspec, b);
                column_add(col, b, one);
            }
#pragma unroll
            for (int u = 0; u < SEG_U; ++u) cur[u] = nxt[u];
            if (++since == SEG_FLUSH_ITERS) {
                regularize_column(col);
                if (__any_sync(FULL, spec_hit(nspec))) {
                    if (spec_hit(nspec)) {
                        seg_rescan(col, body, wstart, it, lane, flags, one);
                        regularize_column(col);
                    }
                }
                nspec = 0;
                since = 0;
                wstart = it + 1;
            }
        }
        // leftover vectors, head and tail: checked adds
        for (uint64_t v = nit * (32 * SEG_U) + lane; v < nvec; v += 32) {
            uint4 q = ldg_stream(body + v);
            column_add_checked(col, q.x, q.y, flags, one);
            column_add_checked(col, q.z, q.w, flags, one);
        }
        if (lane == 0 && head) {
            uint2 q = ldg_one(xs);
            column_add_checked(col, q.x, q.y, flags, one);
        }
        if (lane == 1 && (nbody & 1)) {
            uint2 q = ldg_one(xs + head + 2 * nvec);
            column_add_checked(col, q.x, q.y, flags, one);
        }
        regularize_column(col);
        if (__any_sync(FULL, spec_hit(nspec))) {
            if (spec_hit(nspec) && since) {
                seg_rescan(col, body, wstart, nit - 1, lane, flags, one);
                regularize_column(col);
            }
        }
        __syncwarp();

        // combine the 32 lane columns: |sum| <= 32 (2^51 + 2^11) < 2^57
        const int64_t* wb = win + warp * (D * 32);
        int64_t a0 = 0, a1 = 0;
#pragma unroll 8
        for (int c = 0; c < 32; ++c) {
            int cc = (lane + c) & 31;
            a0 += wb[lane * 32 + cc];
            if (lane + 32 < D) a1 += wb[(lane + 32) * 32 + cc];
        }
        __syncwarp();
        regularize_warp(a0, a1, lane);
        flags = __reduce_or_sync(FULL, flags);
        xsum_result r = finalize_warp(a0, a1, flags, len, canon ? canon + s * XSUM_CANON_LIMBS : nullptr,
                                      su[warp], lane);
        if (lane == 0) {
            out[s] = r.value;
            if (oflags) oflags[s] = r.flags;
        }
    }
}

cudaError_t sum_segments(const double* x, uint64_t nseg, uint64_t seg_len, const uint64_t* offsets, double* out,
                         uint64_t* canon, uint32_t* flags, int num_sms, cudaStream_t s) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_segments, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SEG_SMEM);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    uint64_t want = (nseg + SEG_WARPS - 1) / SEG_WARPS;
    uint64_t cap = (uint64_t)num_sms * 2;   // two 8-warp blocks per SM (86 KB smem each)
    unsigned g = (unsigned)(want < cap ? (want ? want : 1) : cap);
    k_segments<<<g, SEG_WARPS * 32, SEG_SMEM, s>>>(x, nseg, seg_len, offsets, out, canon, flags, 1u, 0xFFFFFFFFu);
    note_launch();
    return cudaGetLastError();
}

}  // namespace xs
