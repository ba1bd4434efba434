// Grid level of the merge tree (§3 step 5 bottom-up; MapReduce
// post-process PAPER.md:1158-1163): every block adds its regularized superaccumulator into a
// grid accumulator in L2 (digit-wise 64-bit atomics: the digits of up to XS_MAXB regularized
// states sum without overflow, and regularizing once at the end gives the same value), and the
// last block to arrive merges it with the handle state and, for a fused one-shot sum, rounds
// (PAPER.md:777-795). Shared by the accumulate kernels.
#pragma once

#include "xsum_device.cuh"
#include "xsum_kernels.h"

namespace xs {

__device__ __forceinline__ int64_t warp_sum64(int64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

// Cross-GPU step of the fused multi-GPU sum (§6.1: the reducers' outputs
// are gathered and merged by the post-process), run by warp 0 of the last block of every rank
// on its rank's final state (b0, b1 regularized digits; fl, cnt): publish the state into slot
// [epoch & 1][rank] of every rank's exchange buffer over NVLink (P2P stores), release-add one to
// every rank's arrival counter, wait (acquire, bounded) until the own counter reaches
// epoch*world, then merge the world slots in rank order with Lemma-1 adds, so
// every rank holds bit-identical digits. A rank can be at most one call ahead of another (it
// needs everyone's contribution to finish a call), hence two slot sets by epoch parity.
// Returns false if the wait timed out (~2 s): the caller flags the result instead of hanging.
__device__ __forceinline__ bool peer_exchange_merge(int64_t& b0, int64_t& b1, uint32_t& fl, uint64_t& cnt,
                                                    const PeerParams& pp, int lane) {
    const uint32_t world = pp.world, rank = pp.rank;
    const size_t set = (size_t)(pp.epoch & 1) * world * XSUM_STATE_BYTES;
    for (uint32_t r = 0; r < world; ++r) {
        xsum_state_image* slot = reinterpret_cast<xsum_state_image*>(pp.bufs[r] + set + (size_t)rank * XSUM_STATE_BYTES);
        slot->digit[lane] = b0;
        if (lane + 32 < D) slot->digit[lane + 32] = b1;
        if (lane == 0) {
            slot->magic = XSUM_MAGIC;
            slot->version = (uint16_t)XSUM_VERSION;
            slot->w = (uint8_t)W;
            slot->ndigits = (uint8_t)D;
            slot->flags = fl;
            slot->reserved = 0;
            slot->count = cnt;
        }
    }
    __threadfence_system();
    __syncwarp();
    bool ok = true;
    if (lane == 0) {
        for (uint32_t r = 0; r < world; ++r) {
            unsigned long long* c = reinterpret_cast<unsigned long long*>(pp.bufs[r] + peer_counter_off(world));
            asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(c) : "memory");
        }
        const unsigned long long* mine =
            reinterpret_cast<const unsigned long long*>(pp.bufs[rank] + peer_counter_off(world));
        const unsigned long long want = pp.epoch * world;
        const long long t0 = clock64();
        unsigned long long v;
        while (true) {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
            if (v >= want) break;
            if (clock64() - t0 > (1ll << 32)) { ok = false; break; }   // ~2 s at 1.9 GHz
            __nanosleep(64);
        }
    }
    ok = __shfl_sync(FULL, ok ? 1 : 0, 0) != 0;
    __syncwarp();
    __threadfence_system();
    int64_t a0 = 0, a1 = 0;
    uint64_t c = 0;
    uint32_t f = 0;
    for (uint32_t r = 0; r < world; ++r) {               // fixed order: identical digits on every rank
        const volatile xsum_state_image* slot =
            reinterpret_cast<const volatile xsum_state_image*>(pp.bufs[rank] + set + (size_t)r * XSUM_STATE_BYTES);
        const int64_t d0 = slot->digit[lane];
        const int64_t d1 = (lane + 32 < D) ? slot->digit[lane + 32] : 0;
        lemma1_add(a0, a1, d0, d1, lane);
        f |= slot->flags;
        c = count_add(c, slot->count, f);
    }
    b0 = a0;
    b1 = a1;
    cnt = c;
    fl = f | (ok ? 0u : XSUM_F_PEER_TIMEOUT);
    return ok;
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
    pdl_wait_predecessor();      // the previous launch may still be merging in the scratch / state
    if (warp == 0) {
        // every block adds its regularized partial into the grid accumulator (L2 atomics,
        // fire-and-forget; |sum| <= XS_MAXB (2^51 + 2^16) < 2^62) and ORs its flags
        asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p.gacc + lane), "l"(a0) : "memory");
        if (lane + 32 < D)
            asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p.gacc + lane + 32), "l"(a1) : "memory");
        if (lane == 0 && bflags) atomicOr(p.gflags, bflags);
        __syncwarp();
        if (lane == 0) {
            // release: this block's adds (ordered before by the warp barrier) are visible to the
            // block that sees the final count; acquire: the last block sees all of them
            uint32_t old;
            asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(p.counter) : "memory");
            *sh_last = (old == (uint32_t)(G - 1));
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) xs_stamp(p.stamps, 3, blockIdx.x);         // arrival atomic returned
    if (!*sh_last) return;
    __threadfence();
    if (warp == 0) {                     // the grid's sum, then the accumulator cleared for the next launch
        red[lane] = __ldcg(p.gacc + lane);
        p.gacc[lane] = 0;
        if (lane + 32 < D) {
            red[lane + 32] = __ldcg(p.gacc + lane + 32);
            p.gacc[lane + 32] = 0;
        }
        if (lane == 0) {
            *sh_flags = __ldcg(p.gflags);
            *p.gflags = 0;
        }
    }
    int64_t st0 = 0, st1 = 0;
    if (warp == 0 && !p.overwrite) {                     // state digits, fetched alongside
        st0 = __ldcg(&p.state->digit[lane]);
        st1 = (lane + 32 < D) ? __ldcg(&p.state->digit[lane + 32]) : 0;
    }
    __syncwarp();
    if (threadIdx.x == 0) xs_stamp(p.stamps, 4, 0);                   // last block: grid sum read
    if (warp == 0) {
        int64_t b0 = red[lane] + st0, b1 = (lane + 32 < D) ? red[lane + 32] + st1 : 0;
        uint32_t fl = *sh_flags;
        uint64_t cnt = n;
        if (!p.overwrite) {
            fl |= p.state->flags;
            cnt = count_add(cnt, p.state->count, fl);
        }
        regularize_warp(b0, b1, lane);
        if (p.peer.bufs) peer_exchange_merge(b0, b1, fl, cnt, p.peer, lane);   // fused multi-GPU step
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
        if (lane == 0) xs_stamp(p.stamps, 5, 0);                      // last block: done
    }
}

}  // namespace xs
