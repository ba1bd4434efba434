// K2: streaming decompose-and-accumulate kernel (the hot path), with the grid-level
// merge of block superaccumulators and an optional fused final rounding.
//
// Design: the paper's in-memory scan (§5: "keep our
// entire superaccumulator stored in internal memory and process the floating-point
// components in any order") with shared memory as the internal memory. Every lane owns a
// private column of D int64 digits (thread-minor layout: digit j of lane l at word
// j*32 + l, so a warp's accesses never bank-conflict whatever the data). Each summand is
// split into two chunks added with carries deferred; a lane column is
// regularized every FLUSH_ELEMS summands. At the end the lane columns
// are summed (warp), the warp sums (block), the block partials (grid: the last block to
// finish, PAPER.md:768-776 bottom-up tree) and the result rounded.
#include <cuda_runtime.h>

#include "grid_tail.cuh"
#include "xsum_device.cuh"
#include "xsum_kernels.h"

namespace xs {

template <int WARPS, int U, int NB, typename E>
struct AccCfg {
    static constexpr int T = WARPS * 32;
    static constexpr int FLUSH_TILES = FLUSH_ELEMS / (Elem<E>::PER_VEC * U);
    static constexpr size_t SMEM = (size_t)WARPS * D * 32 * sizeof(int64_t);
};

template <int U, int T, typename E>
__device__ __noinline__ void rescan_window(int64_t* col, const uint4* body, uint64_t t0, uint64_t t1,
                                              uint64_t G, uint64_t TV, int tid, uint32_t& flags, uint32_t one) {
    // Rare path: this lane summed a NaN/Inf bit pattern as if finite somewhere in tiles
    // [t0, t1] (step G). Re-read its elements and cancel those chunks exactly.
    for (uint64_t tt = t0; tt <= t1; tt += G) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint4 v = ld_stream(body + tt * TV + (uint64_t)u * T + tid);
            Elem<E>::fix_vec(col, v, flags, one);
        }
    }
}

template <int WARPS, int U, int NB, typename E>
__global__ void __launch_bounds__(WARPS * 32, 1)
k_accumulate(const E* x, uint64_t n, AccParams p) {
    using C = AccCfg<WARPS, U, NB, E>;
    using EL = Elem<E>;
    constexpr int PV = EL::PER_VEC;
    constexpr int T = C::T;
    extern __shared__ __align__(16) int64_t win[];
    __shared__ int64_t wsum[WARPS][D];
    __shared__ int64_t su[64];
    __shared__ uint32_t blk_flags;
    __shared__ int is_last;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) xs_stamp(p.stamps, 0, blockIdx.x);                 // block start
    pdl_release_dependents();    // the next launch may take SMs as this grid's blocks finish
    int64_t* col = win + warp * (D * 32) + lane;
#pragma unroll
    for (int j = 0; j < D; ++j) col[j * 32] = 0;
    if (tid == 0) blk_flags = 0;
    uint32_t flags = 0;
    pdl_wait_predecessor();      // inputs are read only after the preceding launch completed
    if (p.skip && *(volatile const uint32_t*)p.skip) return;     // K12: an earlier iteration stopped

    // peel up to PV-1 head elements to reach 16-B alignment; <= PV-1 tail elements remain
    uint64_t head = ((16 - ((uintptr_t)x & 15)) & 15) / sizeof(E);
    if (head > n) head = n;
    const uint64_t nbody = n - head;
    const uint64_t nvec = nbody / PV;
    const uint4* body = reinterpret_cast<const uint4*>(x + head);
    const uint64_t TV = (uint64_t)T * U;
    const uint64_t ntiles = nvec / TV;
    const uint64_t G = gridDim.x;

    const uint32_t one = p.one, mone = p.mone;
    uint32_t nspec = 0;                 // NaN/Inf patterns summed unchecked in this window
    uint64_t wstart = blockIdx.x, tlast = 0;
    bool any_tile = false;
    auto load_tile = [&](uint4 (&buf)[U], uint64_t tt) {
        if (tt < ntiles) {
#pragma unroll
            for (int u = 0; u < U; ++u) buf[u] = ld_stream(body + tt * TV + (uint64_t)u * T + tid);
        }
    };
    // NB register buffers of U vectors rotate without moves (the unrolled b loop indexes them
    // statically): while one tile is decoded the next NB-1 are in flight. The window check
    // runs once per NB-tile group, outside the unrolled loop, and inlines the regularization:
    // an out-of-line call here would have to save the in-flight buffers, i.e. wait for them.
    constexpr int GROUPS_PER_WINDOW = C::FLUSH_TILES / NB;    // window = NB*GROUPS <= FLUSH_TILES tiles
    uint4 buf[NB][U];
    uint64_t t = blockIdx.x;
#pragma unroll
    for (int b = 0; b < NB; ++b) load_tile(buf[b], t + (uint64_t)b * G);
    bool more = t < ntiles;
    int groups = 0;
    while (more) {
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            if (more) {
#pragma unroll
                for (int u = 0; u < U; ++u) EL::add_vec(col, buf[b][u], nspec, one, mone);
                any_tile = true;
                tlast = t;
                load_tile(buf[b], t + (uint64_t)NB * G);
                t += G;
                more = t < ntiles;
            }
        }
        if (++groups == GROUPS_PER_WINDOW) {
            regularize_column_inl(col);
            if (__any_sync(FULL, EL::hit(nspec))) {        // rare: cancel NaN/Inf patterns
                if (EL::hit(nspec)) {
                    rescan_window<U, T, E>(col, body, wstart, tlast, G, TV, tid, flags, one);
                    regularize_column(col);
                }
            }
            nspec = 0;
            groups = 0;
            wstart = t;
            any_tile = false;
        }
    }

    // leftover vectors (< one tile), the unaligned head and the tail elements: checked adds by
    // the block that would own the next tile.
    bool touched = blockIdx.x < ntiles;                 // every thread takes part in every tile
    if (blockIdx.x == ntiles % G) {
        const uint64_t v0 = ntiles * TV;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint64_t v = v0 + (uint64_t)u * T + tid;
            if (v < nvec) {
                EL::add_vec_checked(col, ld_stream(body + v), flags, one);
                touched = true;
            }
        }
        const uint64_t tail = nbody - nvec * PV;
        if ((uint64_t)tid < head) {
            EL::add_one_checked(col, x + tid, flags, one);
            touched = true;
        }
        if (tid >= PV && (uint64_t)(tid - PV) < tail) {
            EL::add_one_checked(col, x + head + nvec * PV + (tid - PV), flags, one);
            touched = true;
        }
    }
    if (tid == 0) xs_stamp(p.stamps, 1, blockIdx.x);                 // stream done
    if (__any_sync(FULL, EL::hit(nspec))) {
        if (EL::hit(nspec) && any_tile) {
            regularize_column(col);
            rescan_window<U, T, E>(col, body, wstart, tlast, G, TV, tid, flags, one);
        }
    }
    __syncwarp();

    // warp: sum the 32 raw lane columns into regularized digits (lane l holds digits l and
    // l+32; rotated reads keep the 32 lanes on 32 distinct columns). A warp that added nothing
    // (small inputs) has zero columns and skips the combine.
    {
        int64_t s0 = 0, s1 = 0;
        if (__any_sync(FULL, touched)) combine_raw_columns(win + warp * (D * 32), s0, s1, lane);
        wsum[warp][lane] = s0;
        if (lane + 32 < D) wsum[warp][lane + 32] = s1;
        uint32_t f = __reduce_or_sync(FULL, flags);
        if (lane == 0 && f) atomicOr(&blk_flags, f);
    }
    __syncthreads();
    if (tid == 0) xs_stamp(p.stamps, 2, blockIdx.x);                 // warp combines done

    // block: sum the warp partials (|.| <= WARPS*(2^51+2^16) < 2^56), regularize, publish;
    // the last block merges the grid (grid_tail.cuh).
    int64_t a0 = 0, a1 = 0;
    if (warp == 0) {
#pragma unroll
        for (int w = 0; w < WARPS; ++w) {
            a0 += wsum[w][lane];
            if (lane + 32 < D) a1 += wsum[w][lane + 32];
        }
        regularize_warp(a0, a1, lane);
    }
    grid_tail<WARPS>(a0, a1, blk_flags, n, p, wsum[0], su, &blk_flags, &is_last, warp, lane);
}

template <int WARPS, int U, int NB, typename E>
static cudaError_t launch_accumulate(const E* x, uint64_t n, const AccParams& p, int num_sms, cudaStream_t s) {
    using C = AccCfg<WARPS, U, NB, E>;
    static unsigned long long smem_set = 0;
    if (cudaError_t e = ensure_smem(k_accumulate<WARPS, U, NB, E>, C::SMEM, smem_set)) return e;
    uint64_t head = ((16 - ((uintptr_t)x & 15)) & 15) / sizeof(E);
    if (head > n) head = n;
    const uint64_t ntiles = ((n - head) / Elem<E>::PER_VEC) / ((uint64_t)C::T * U);
    uint64_t g = ntiles < (uint64_t)num_sms ? ntiles : (uint64_t)num_sms;
    if (g < 1) g = 1;
    if (g > XS_MAXB) g = XS_MAXB;
    cudaError_t e = launch_pdl(n * sizeof(E) < PDL_MAX_BYTES, k_accumulate<WARPS, U, NB, E>, (unsigned)g, C::T, C::SMEM, s, x, n, p);
    note_launch();
    return e;
}

#ifndef XS_ACC_WARPS
#define XS_ACC_WARPS 16   // 16 warps x 42 digits x 32 lanes x 8 B = 168 KiB of lane columns per SM
#endif
#ifndef XS_ACC_U
#define XS_ACC_U 4        // 16-B vectors per thread per tile
#endif
#ifndef XS_ACC_NB
#define XS_ACC_NB 5       // rotating register buffers (NB-1 tiles in flight); tools/variants.py:
#endif                    // c2 671 (NB=3), 708 (4), 715 G/s (5) at U=4

cudaError_t accumulate(const double* x, uint64_t n, const AccParams& p, int num_sms, cudaStream_t s) {
    return launch_accumulate<XS_ACC_WARPS, XS_ACC_U, XS_ACC_NB, double>(x, n, p, num_sms, s);
}


}  // namespace xs
