// K12: the condition-number-sensitive summation (§4).
//
// The paper's iteration: r = 2, then r <- r^2; each iteration sums the n values bottom-up over a
// summation tree with r-truncated sparse superaccumulators - every internal
// node is the truncated Lemma-1 sum (Lemma 2 :859-872) of its
// children - and stops when a stopping condition holds for the rounded root,
// or when nothing was truncated. r = 256 > 42 digits never truncates: that iteration is the
// exact dense sum (K2), whose value is the same exact sum.
//
// Tree (reading C2): the complete binary tree over the index order; node (L, j) covers
// [j 2^L, (j+1) 2^L) and a node without a right child is its left child. The GPU evaluates it
// level by level in aligned power-of-two chunks: a thread builds the subtree of its 2^G leaves
// from registers (static recursion), a warp the next 5 levels by shuffles, a block the next
// log2(warps) levels through shared memory; block roots go to a record array that the next pass
// treats as leaves, until one root is left. Every node therefore sees exactly the oracle's
// operands, so the root digits match the oracle bit for bit.
//
// A sparse superaccumulator here is a sorted list of <= RC entries (index, regularized digit),
// indices descending, unused slots index -1 (registers; RC = r). eps_min (reading C3): every
// truncating node records the index of its least significant kept entry; the iteration's E_cut
// is the maximum over all nodes (atomicMax), so |S - T| < n R^E_cut 2^-1074.
#include <cuda_runtime.h>

#include "xsum_device.cuh"
#include "xsum_kernels.h"

namespace xs {
namespace cs {

// control block at the start of the work buffer
struct Ctl {
    uint32_t done;        // 1 once an iteration stopped (later launches of the call exit at entry)
    int32_t e_cut;        // this iteration's max truncation index (-1: none), reset by k_cs_final
    uint32_t flags;       // NaN / +-Inf seen (leaves)
    uint32_t pad;
};
constexpr size_t CTL_BYTES = 256;
constexpr size_t ZERO_ROOT_OFF = 64;                                 // 16 zero records: the empty tree's root
constexpr size_t STATE_OFF = CTL_BYTES;                              // 384-byte state (exact pass)
constexpr size_t SCRATCH_OFF = 1024;                                 // K2 scratch, 256-aligned
constexpr size_t RECS_OFF = SCRATCH_OFF + ((SCRATCH_BYTES + 255) / 256) * 256;

template <int RC>
struct SSA {
    int k[RC];          // digit index, descending; -1 = unused
    int64_t v[RC];      // regularized digit (|v| <= R-1), non-zero where k >= 0
};

template <int RC>
__device__ __forceinline__ void ssa_clear(SSA<RC>& a) {
#pragma unroll
    for (int j = 0; j < RC; ++j) { a.k[j] = -1; a.v[j] = 0; }
}

// Step 2: x -> at most two entries, +-hi at index i+1 and +-lo at index i,
// M 2^o = hi R + lo (0 <= lo, hi < R), |x| = M 2^(k-1074), i = k / 52, o = k mod 52.
template <int RC>
__device__ __forceinline__ void ssa_leaf(SSA<RC>& a, uint64_t b, uint32_t& flags) {
    ssa_clear(a);
    const uint32_t e = (uint32_t)(b >> 52) & 0x7FF;
    const uint64_t m = b & MASK;
    if (e == 0x7FF) {
        flags |= m ? XSUM_F_NAN : ((b >> 63) ? XSUM_F_NINF : XSUM_F_PINF);
        return;
    }
    const uint64_t M = m | ((uint64_t)(e != 0) << 52);
    const uint32_t k = (e ? e : 1) - 1;
    const int i = (int)(k / 52), o = (int)(k % 52);
    const uint64_t lo = (M << o) & MASK;
    const uint64_t hi = o ? (M >> (52 - o)) : (M >> 52);
    const bool neg = b >> 63;
    const int64_t slo = neg ? -(int64_t)lo : (int64_t)lo, shi = neg ? -(int64_t)hi : (int64_t)hi;
    static_assert(RC >= 2, "a leaf has up to two entries");
    // descending: hi first when present
    if (hi) {
        a.k[0] = i + 1; a.v[0] = shi;
        if (lo) { a.k[1] = i; a.v[1] = slo; }
    } else if (lo) {
        a.k[0] = i; a.v[0] = slo;
    }
}

__device__ __forceinline__ void ce_desc(int& ka, int64_t& va, int& kb, int64_t& vb) {
    const bool sw = kb > ka;
    const int tk = sw ? kb : ka;
    kb = sw ? ka : kb;
    ka = tk;
    const int64_t tv = sw ? vb : va;
    vb = sw ? va : vb;
    va = tv;
}

// The r-truncated Lemma-1 sum of two sparse superaccumulators (PAPER.md:703-711, :559-628,
// :721-725). cut := max(cut, index of the least significant kept entry) if entries were dropped.
// r >= XS_CS_SLOTS: the selection of the RC most significant entries scatters the candidates by
// rank into per-thread shared-memory slots instead of an RC x 2U select network (r = 4: c2 step
// 16.38 -> 15.29 ms; r = 2 is faster with the selects; profiles/r02_condsens.txt)
#ifndef XS_CS_SLOTS
#define XS_CS_SLOTS 4
#endif
template <int RC>
__device__ __forceinline__ void ssa_merge(SSA<RC>& a, const SSA<RC>& b, int& cut, int64_t* slot, int sstride) {
    constexpr int U = 2 * RC;
    int k[U];
    int64_t p[U];
    // A descending ++ B reversed (ascending) is bitonic; a bitonic merge sorts it descending
#pragma unroll
    for (int j = 0; j < RC; ++j) {
        k[j] = a.k[j]; p[j] = a.v[j];
        k[U - 1 - j] = b.k[j]; p[U - 1 - j] = b.v[j];
    }
#pragma unroll
    for (int s = RC; s >= 1; s >>= 1) {
#pragma unroll
        for (int j = 0; j < U; ++j)
            if ((j & s) == 0) ce_desc(k[j], p[j], k[j + s], p[j + s]);
    }
    // P_i = Y_i + Z_i on the merged active indices: an index occurs at most twice, adjacently;
    // the second occurrence becomes dead (-2)
#pragma unroll
    for (int j = 0; j + 1 < U; ++j) {
        const bool dup = k[j] >= 0 && k[j] == k[j + 1];
        p[j] = dup ? p[j] + p[j + 1] : p[j];
        p[j + 1] = dup ? 0 : p[j + 1];
        k[j + 1] = dup ? -2 : k[j + 1];
    }
    // signed carries C_{i+1} of Lemma 1 and W_i = P_i - C_{i+1} R
    int c[U];
    int64_t s[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
        c[j] = lemma1_carry(p[j]);                 // 0 for dead / unused entries (p = 0)
        s[j] = p[j] - (int64_t)c[j] * R;
    }
    // S_i = W_i + C_i: the carry into index i comes from the next live entry if its index is i-1
    // (at j+1, or at j+2 when j+1 is this entry's dead duplicate)
    int64_t sv[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
        int cin = 0;
        if (j + 1 < U && k[j + 1] == k[j] - 1) cin += c[j + 1];
        if (j + 2 < U && k[j + 1] == -2 && k[j + 2] == k[j] - 1) cin += c[j + 2];
        sv[j] = s[j] + cin;
    }
    // candidate entries in descending index order: the carry out of entry j when no live entry
    // holds index k_j + 1 (it becomes a new active index), then entry j itself if non-zero
    int ck[2 * U];
    int64_t cv[2 * U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
        bool absorbed = false;
        if (j >= 1 && k[j - 1] == k[j] + 1) absorbed = true;
        if (j >= 2 && k[j - 1] == -2 && k[j - 2] == k[j] + 1) absorbed = true;
        const bool orphan = k[j] >= 0 && c[j] != 0 && !absorbed;
        ck[2 * j] = orphan ? k[j] + 1 : -1;
        cv[2 * j] = orphan ? (int64_t)c[j] : 0;
        const bool live = k[j] >= 0 && sv[j] != 0;
        ck[2 * j + 1] = live ? k[j] : -1;
        cv[2 * j + 1] = live ? sv[j] : 0;
    }
    // keep the RC most significant non-zero entries
    int cnt = 0;
    static_assert(RC <= 4, "r = 16 uses the warp-dense kernel");
#if XS_CS_SLOTS
    if (slot) {            // scatter the first RC by rank into this thread's shared slots
        uint32_t nzm = 0;
#pragma unroll
        for (int t = 0; t < 2 * U; ++t) nzm |= (uint32_t)(ck[t] >= 0) << t;
        cnt = __popc(nzm);
#pragma unroll
        for (int t = 0; t < 2 * U; ++t) {
            const int rank = __popc(nzm & ((1u << t) - 1));
            if (ck[t] >= 0 && rank < RC) slot[rank * sstride] = (int64_t)(((uint64_t)cv[t] << 6) | (uint64_t)ck[t]);
        }
#pragma unroll
        for (int q = 0; q < RC; ++q) {
            const int64_t r = q < cnt ? slot[q * sstride] : 0;
            a.k[q] = r ? (int)(r & 63) : -1;
            a.v[q] = r >> 6;
        }
    } else
#endif
    {
        ssa_clear(a);
#pragma unroll
        for (int t = 0; t < 2 * U; ++t) {
            const bool nz = ck[t] >= 0;
#pragma unroll
            for (int q = 0; q < RC; ++q) {
                const bool hit = nz && cnt == q;
                a.k[q] = hit ? ck[t] : a.k[q];
                a.v[q] = hit ? cv[t] : a.v[q];
            }
            cnt += nz;
        }
    }
    if (cnt > RC) cut = max(cut, a.k[RC - 1]);
}

// Code size: the first version inlined a merge at every node of a static recursion over the 2^G
// leaves (~64 KB of SASS per kernel; ncu: no_instruction stalls 3.4 per issue, the L1.5 I-cache is
// 32 KB). The binary counter below has G merge sites in its loop body; an out-of-line merge
// measured no faster (r = 2: 5.73 vs 5.54 ms, r = 4: 13.9 vs 14.0 ms for 2^28 leaves;
// profiles/r02_condsens.txt).
template <int RC>
__device__ __forceinline__ void merge_into(SSA<RC>& a, const SSA<RC>& b, int& cut, int64_t* slot = nullptr,
                                           int sstride = 0) {
    ssa_merge(a, b, cut, slot, sstride);
}

// records: (digit << 6) | index, 0 = unused slot (the sparse image record format, include/xsum.h)
template <int RC>
__device__ __forceinline__ void ssa_load(SSA<RC>& a, const int64_t* rec) {
#pragma unroll
    for (int j = 0; j < RC; ++j) {
        const int64_t r = rec[j];
        a.k[j] = r ? (int)(r & 63) : -1;
        a.v[j] = r >> 6;
    }
}
template <int RC>
__device__ __forceinline__ void ssa_store(const SSA<RC>& a, int64_t* rec) {
#pragma unroll
    for (int j = 0; j < RC; ++j) rec[j] = a.k[j] >= 0 ? (int64_t)(((uint64_t)a.v[j] << 6) | (uint64_t)a.k[j]) : 0;
}
template <int RC>
__device__ __forceinline__ void ssa_shfl_down(SSA<RC>& o, const SSA<RC>& a, int d) {
#pragma unroll
    for (int j = 0; j < RC; ++j) {
        o.k[j] = __shfl_down_sync(FULL, a.k[j], d);
        o.v[j] = __shfl_down_sync(FULL, a.v[j], d);
    }
}

#ifndef XS_CS2_G
#define XS_CS2_G 6
#endif
#ifndef XS_CS4_G
#define XS_CS4_G 4
#endif
#ifndef XS_CS4_MINB
#define XS_CS4_MINB 2
#endif
template <int RC> struct Shape;
template <> struct Shape<2> { static constexpr int G = XS_CS2_G, T = 256, MINB = 2; };
template <> struct Shape<4> { static constexpr int G = XS_CS4_G, T = 256, MINB = XS_CS4_MINB; };
// r = 16: a sorted 16-entry list per thread does not fit in registers (spills, ~0.9 us per
// node); that iteration keeps the superaccumulator dense across a warp instead (k_cs_tree_w16)
constexpr int W16_WARPS = 8, W16_LOG = 10;      // 2^10 consecutive leaves per warp chunk
template <int RC>
constexpr int chunk_log2() {
    if constexpr (RC == 16) return W16_LOG;
    else return Shape<RC>::G + (Shape<RC>::T == 256 ? 8 : 7);
}

// One pass: chunk c (2^B consecutive leaves, B = G + log2 T) -> its subtree root, recs_out[c].
template <int RC, bool DOUBLES>
__global__ void __launch_bounds__(Shape<RC>::T, Shape<RC>::MINB)
k_cs_tree(const void* __restrict__ src, uint64_t nleaf, int64_t* __restrict__ recs_out, uint64_t nchunks, Ctl* ctl) {
    constexpr int G = Shape<RC>::G, T = Shape<RC>::T, NL = 1 << G, WARPS = T / 32;
    constexpr int B = chunk_log2<RC>();
    __shared__ int64_t wroot[WARPS][RC];
    __shared__ int wpres[WARPS];
#if XS_CS_SLOTS
    __shared__ int64_t cslot[RC * T];                 // per-thread compaction slots, stride T
#endif
    if (*(volatile uint32_t*)&ctl->done) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#if XS_CS_SLOTS
    int64_t* const slot = (RC >= XS_CS_SLOTS) ? cslot + tid : nullptr;
#else
    int64_t* const slot = nullptr;
#endif
    int cut = -1;
    uint32_t flags = 0;
    for (uint64_t chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
        const uint64_t first = (chunk << B) + ((uint64_t)tid << G);
        const int nleft = first < nleaf ? (int)min((uint64_t)NL, nleaf - first) : 0;
        // this thread's 2^G leaves: the complete subtree by a binary counter (reading C2): after
        // leaf p, the subtrees of sizes 2^L that end at p are summed with their left siblings
        // (stack[L]) while bit L of p is set; a partial last group folds the pending stack
        // entries from the smallest subtree up (a missing right child passes its left child up)
        SSA<RC> a;
        ssa_clear(a);
        if (nleft > 0) {
            SSA<RC> stack[G];
#pragma unroll 1
            for (int p = 0; p < nleft; ++p) {
                SSA<RC> cur;
                if constexpr (DOUBLES)
                    ssa_leaf(cur, static_cast<const uint64_t*>(src)[first + p], flags);
                else
                    ssa_load(cur, static_cast<const int64_t*>(src) + (first + p) * RC);
                bool carry = true;
#pragma unroll
                for (int L = 0; L < G; ++L) {
                    if (carry) {
                        if ((p >> L) & 1) {
                            merge_into(cur, stack[L], cut, slot, T);
                        } else {
                            stack[L] = cur;
                            carry = false;
                        }
                    }
                }
                if (carry) a = cur;                 // p = 2^G - 1: the whole group
            }
            if (nleft < NL) {
                bool have = false;
#pragma unroll
                for (int L = 0; L < G; ++L) {
                    if ((nleft >> L) & 1) {
                        if (have) merge_into(a, stack[L], cut, slot, T);
                        else a = stack[L];
                        have = true;
                    }
                }
            }
        }
        bool pres = nleft > 0;
        // warp levels G .. G+4 (lane pairs by shuffles)
#pragma unroll 1
        for (int d = 1; d < 32; d <<= 1) {
            SSA<RC> b;
            ssa_shfl_down(b, a, d);
            const bool bpres = __shfl_down_sync(FULL, pres, d);
            if ((lane & (2 * d - 1)) == 0 && bpres) merge_into(a, b, cut, slot, T);
        }
        if (lane == 0) {
            ssa_store(a, wroot[warp]);
            wpres[warp] = pres;
        }
        __syncthreads();
        // block levels (the warps' roots)
        if (warp == 0) {
            SSA<RC> w;
            ssa_clear(w);
            bool wp = false;
            if (lane < WARPS) {
                ssa_load(w, wroot[lane]);
                wp = wpres[lane];
            }
#pragma unroll 1
            for (int d = 1; d < WARPS; d <<= 1) {
                SSA<RC> b;
                ssa_shfl_down(b, w, d);
                const bool bpres = __shfl_down_sync(FULL, wp, d);
                if ((lane & (2 * d - 1)) == 0 && bpres) merge_into(w, b, cut, slot, T);
            }
            if (lane == 0) ssa_store(w, recs_out + chunk * RC);
        }
        __syncthreads();
    }
    // this iteration's E_cut and the special-value flags
#pragma unroll
    for (int d = 16; d; d >>= 1) cut = max(cut, __shfl_xor_sync(FULL, cut, d));
    const uint32_t f = __reduce_or_sync(FULL, flags);
    if (lane == 0) {
        if (cut >= 0) atomicMax(&ctl->e_cut, cut);
        if (f) atomicOr(&ctl->flags, f);
    }
}

// ---------------------------------------------------------------------------------------------
// r = 16: the same tree with the superaccumulator dense across a warp - lane l holds digits l and
// l + 32, as in the exact path (a0, a1). The r-truncated Lemma-1 sum is lemma1_add (PAPER.md:
// 578-628; identical to the sparse sum: an absent index is a zero digit, which only a carry
// makes non-zero) followed by keeping the 16 most significant non-zero digits (two ballots). Each
// warp walks its chunk of 2^W16_LOG leaves in order with a binary counter whose pending subtree
// roots live in shared memory; a merge costs ~60 warp instructions (lemma1_add ~35, the truncation
// test, the stack) instead of a 16-entry sorted merge per thread. The leaves of a 32-leaf step are
// decomposed once, lane j taking leaf j, and broadcast by shuffles (ncu: every lane decoding every
// leaf was ~60 of ~150 warp instructions per leaf; c3 step 63.6 -> 50.0 ms).
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void trunc_dense(int64_t& a0, int64_t& a1, int r, int& cut, int lane) {
    const uint32_t lo = __ballot_sync(FULL, a0 != 0);
    const uint32_t hi = __ballot_sync(FULL, a1 != 0);
    const uint64_t m = ((uint64_t)hi << 32) | lo;
    if (__popcll(m) > r) {                               // warp-uniform
        uint64_t mm = m;
        for (int q = 1; q < r; ++q) mm &= ~(1ull << (63 - __clzll(mm)));   // drop the top r-1
        const int j = 63 - __clzll(mm);                  // the r-th most significant non-zero digit
        if (lane < j) a0 = 0;
        if (lane + 32 < j) a1 = 0;
        cut = max(cut, j);
    }
}

// the two entries of one leaf x (bit pattern b): +-lo at digit i, +-hi at i+1;
// i = -1 for NaN / Inf (flagged, summed as zero)
__device__ __forceinline__ void leaf_parts(uint64_t b, int& i, int64_t& slo, int64_t& shi, uint32_t& flags) {
    i = -1;
    slo = shi = 0;
    const uint32_t e = (uint32_t)(b >> 52) & 0x7FF;
    const uint64_t m = b & MASK;
    if (e == 0x7FF) {
        flags |= m ? XSUM_F_NAN : ((b >> 63) ? XSUM_F_NINF : XSUM_F_PINF);
        return;
    }
    const uint64_t M = m | ((uint64_t)(e != 0) << 52);
    const uint32_t k = (e ? e : 1) - 1;
    i = (int)(k / 52);
    const int o = (int)(k % 52);
    const uint64_t lo = (M << o) & MASK;
    const uint64_t hi = o ? (M >> (52 - o)) : (M >> 52);
    const bool neg = b >> 63;
    slo = neg ? -(int64_t)lo : (int64_t)lo;
    shi = neg ? -(int64_t)hi : (int64_t)hi;
}

// dense digits of leaf j of the warp's 32 (lane j decomposed it: li / llo / lhi), in every lane
__device__ __forceinline__ void dense_leaf_from(int li, int64_t llo, int64_t lhi, int j, int64_t& a0, int64_t& a1,
                                                int lane) {
    const int i = __shfl_sync(FULL, li, j);
    const int64_t slo = __shfl_sync(FULL, llo, j), shi = __shfl_sync(FULL, lhi, j);
    a0 = lane == i ? slo : (lane == i + 1 ? shi : 0);
    a1 = lane + 32 == i ? slo : (lane + 32 == i + 1 ? shi : 0);
}

// a 16-record leaf (a previous pass's chunk root) to dense digits
__device__ __forceinline__ void dense_from_records(const int64_t* rec, int64_t& a0, int64_t& a1, int lane) {
    const int64_t mine = lane < 16 ? rec[lane] : 0;
    a0 = a1 = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const int64_t r = __shfl_sync(FULL, mine, q);
        const int k = r ? (int)(r & 63) : -1;
        if (k == lane) a0 = r >> 6;
        if (k == lane + 32) a1 = r >> 6;
    }
}

// dense digits (at most 16 non-zero) to 16 records in descending index order, zero padded
__device__ __forceinline__ void dense_to_records(int64_t a0, int64_t a1, int64_t* rec, int lane) {
    const uint32_t lo = __ballot_sync(FULL, a0 != 0);
    const uint32_t hi = __ballot_sync(FULL, a1 != 0);
    const uint64_t m = ((uint64_t)hi << 32) | lo;
    const int nnz = __popcll(m);
    if (a0 != 0) {
        const int rank = __popcll(m >> (lane + 1));
        if (rank < 16) rec[rank] = (int64_t)(((uint64_t)a0 << 6) | (uint64_t)lane);
    }
    if (a1 != 0) {
        const int pos = lane + 32;
        const int rank = __popcll(m >> (pos + 1));
        if (rank < 16) rec[rank] = (int64_t)(((uint64_t)a1 << 6) | (uint64_t)pos);
    }
    if (lane >= nnz && lane < 16) rec[lane] = 0;
}

template <bool DOUBLES>
__global__ void __launch_bounds__(W16_WARPS * 32)
k_cs_tree_w16(const void* __restrict__ src, uint64_t nleaf, int64_t* __restrict__ recs_out, uint64_t nchunks,
              Ctl* ctl) {
    constexpr int R16 = 16, NLW = 1 << W16_LOG;
    __shared__ int64_t stk[W16_WARPS][W16_LOG][64];      // pending subtree roots (dense digits)
    if (*(volatile uint32_t*)&ctl->done) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t* const st = &stk[warp][0][0];
    int cut = -1;
    uint32_t flags = 0;
    const uint64_t nw = (uint64_t)gridDim.x * W16_WARPS;
    for (uint64_t chunk = (uint64_t)blockIdx.x * W16_WARPS + warp; chunk < nchunks; chunk += nw) {
        const uint64_t first = chunk << W16_LOG;
        const int nleft = (int)min((uint64_t)NLW, nleaf - first);
        int64_t a0 = 0, a1 = 0;                          // the chunk root
        for (int base = 0; base < nleft; base += 32) {
            // lane j decomposes leaf base + j once (instead of every lane redoing each leaf)
            int li = -1;
            int64_t llo = 0, lhi = 0;
            if constexpr (DOUBLES) {
                if (base + lane < nleft)
                    leaf_parts(static_cast<const uint64_t*>(src)[first + base + lane], li, llo, lhi, flags);
            }
            const int cnt = min(32, nleft - base);
            for (int j = 0; j < cnt; ++j) {
                const int p = base + j;
                int64_t c0, c1;
                if constexpr (DOUBLES)
                    dense_leaf_from(li, llo, lhi, j, c0, c1, lane);
                else
                    dense_from_records(static_cast<const int64_t*>(src) + (first + p) * R16, c0, c1, lane);
                // binary counter (reading C2): sum with the left siblings while bit L of p is set
                int L = 0;
                while (L < W16_LOG && ((p >> L) & 1)) {
                    lemma1_add(c0, c1, st[L * 64 + lane], st[L * 64 + 32 + lane], lane);
                    trunc_dense(c0, c1, R16, cut, lane);
                    ++L;
                }
                if (L < W16_LOG) {
                    st[L * 64 + lane] = c0;
                    st[L * 64 + 32 + lane] = c1;
                } else {
                    a0 = c0;
                    a1 = c1;
                }
            }
        }
        if (nleft < NLW) {                                // fold the pending roots, smallest first
            bool have = false;
            for (int L = 0; L < W16_LOG; ++L) {
                if ((nleft >> L) & 1) {
                    const int64_t s0 = st[L * 64 + lane], s1 = st[L * 64 + 32 + lane];
                    if (have) {
                        lemma1_add(a0, a1, s0, s1, lane);
                        trunc_dense(a0, a1, R16, cut, lane);
                    } else {
                        a0 = s0;
                        a1 = s1;
                    }
                    have = true;
                }
            }
        }
        dense_to_records(a0, a1, recs_out + chunk * R16, lane);
        __syncwarp();
    }
    const uint32_t f = __reduce_or_sync(FULL, flags);
    if (lane == 0) {
        if (cut >= 0) atomicMax(&ctl->e_cut, cut);
        if (f) atomicOr(&ctl->flags, f);
    }
}

// RN(y (+) d) == y for d = n 2^a and the gap 2^g on one side of y (round to nearest, ties to
// even; `odd` = y's significand is odd): d < 2^(g-1), or d == 2^(g-1) and y even.
__device__ __forceinline__ bool stays(uint64_t n, int a, int g, bool odd) {
    const int s = g - 1 - a;                      // compare n with 2^s
    if (s < 0) return false;                      // n 2^a >= 2^a > 2^(g-1)
    if (s >= 64) return true;
    const uint64_t h = s == 63 ? (1ull << 63) : (1ull << s);
    return n < h || (n == h && !odd);
}

// Stopping conditions (readings C3, C4) for the finite non-zero y.
__device__ __forceinline__ bool stop_ok(uint64_t ybits, uint64_t n, int e_cut, int rule) {
    const uint32_t e = (uint32_t)(ybits >> 52) & 0x7FF;
    const uint64_t m = ybits & MASK;
    if (e == 0x7FF || (e == 0 && m == 0)) return false;
    const int ue = (int)(e ? e : 1) - 1075;       // exponent of y's least significant bit
    const int a = 52 * e_cut - 1074;              // eps_min = 2^a
    if (rule == 2) {
        const int clog = 64 - __clzll(n - 1);     // ceil(log2 n) for n >= 1
        return ue >= a + clog + 2;
    }
    const int g_up = ue;                          // gap away from zero
    const int g_dn = (m == 0 && e > 1) ? ue - 1 : ue;   // gap toward zero (smaller below a power of two)
    const bool odd = m & 1;
    return stays(n, a, g_up, odd) && stays(n, a, g_dn, odd);
}

// End of an iteration (one warp): the root's value rounded (PAPER.md:777-795 via finalize_warp),
// the stopping decision, and on stop the outputs.
template <int RC>
__global__ void k_cs_final(const int64_t* __restrict__ root, uint64_t n, int r, int iteration, int rule, Ctl* ctl,
                           xsum_result* res, xsum_condsens_info* info, uint64_t* canon) {
    __shared__ int64_t su[64];
    const int lane = threadIdx.x & 31;
    if (*(volatile uint32_t*)&ctl->done) return;
    int64_t a0 = 0, a1 = 0;
    int nnz = 0;
#pragma unroll
    for (int j = 0; j < RC; ++j) {
        const int64_t rr = root[j];
        if (rr) {
            ++nnz;
            const int k = (int)(rr & 63);
            if (k == lane) a0 = rr >> 6;
            if (k == lane + 32) a1 = rr >> 6;
        }
    }
    const int e_cut = ctl->e_cut;
    const uint32_t flags = ctl->flags;
    const xsum_result fin = finalize_warp(a0, a1, 0u, n, nullptr, su, lane);   // y: the finite root
    uint64_t ybits = __double_as_longlong(fin.value);
    ybits = __shfl_sync(FULL, ybits, 0);
    const bool stop = e_cut < 0 || stop_ok(ybits, n, e_cut, rule);
    if (stop) {
        const xsum_result out = finalize_warp(a0, a1, flags, n, canon, su, lane);
        if (lane == 0) {
            *res = out;
            info->r = (uint32_t)r;
            info->iterations = (uint32_t)iteration;
            info->e_cut = e_cut;
            info->exact = e_cut < 0;
            info->rule = (uint32_t)rule;
            info->nnz = (uint32_t)nnz;
        }
        if (lane < 16) info->root[lane] = lane < RC ? (uint64_t)root[lane] : 0;
    }
    __syncwarp();
    if (lane == 0) {
        ctl->e_cut = -1;                      // the next iteration's maximum starts empty
        ctl->flags = 0;
        if (stop) ctl->done = 1;
    }
}

// start of a call: control block, and the exact pass's K2 scratch (arrival counter, grid flags,
// grid accumulator) zeroed - every K2 launch leaves it zeroed again
__global__ void k_cs_init(Ctl* ctl, uint8_t* scratch, int nwords) {
    if (threadIdx.x == 0) {
        ctl->done = 0;
        ctl->e_cut = -1;
        ctl->flags = 0;
    }
    if (threadIdx.x < 16) reinterpret_cast<int64_t*>(reinterpret_cast<uint8_t*>(ctl) + ZERO_ROOT_OFF)[threadIdx.x] = 0;
    for (int i = threadIdx.x; i < nwords; i += blockDim.x) reinterpret_cast<uint64_t*>(scratch)[i] = 0;
}

// After the exact pass (r = 256, K2 with skip = done): record it if it ran.
__global__ void k_cs_exact_info(Ctl* ctl, int rule, xsum_condsens_info* info) {
    const int lane = threadIdx.x;
    if (*(volatile uint32_t*)&ctl->done) return;
    if (lane == 0) {
        info->r = 256;
        info->iterations = 4;
        info->e_cut = -1;
        info->exact = 1;
        info->rule = (uint32_t)rule;
        info->nnz = 0;
        ctl->done = 1;
    }
    if (lane < 16) info->root[lane] = 0;
}

template <int RC>
uint64_t pass_count(uint64_t m) {
    constexpr int B = chunk_log2<RC>();
    return (m + (1ull << B) - 1) >> B;
}

template <int RC>
size_t recs_bytes(uint64_t n, size_t& second) {
    const uint64_t m1 = pass_count<RC>(n);
    const uint64_t m2 = m1 > 1 ? pass_count<RC>(m1) : 0;
    second = (size_t)m2 * RC * 8;
    return (size_t)m1 * RC * 8;
}

template <int RC>
cudaError_t iteration(const double* x, uint64_t n, int iter, int rule, uint8_t* work, size_t first_bytes,
                      xsum_result* res, xsum_condsens_info* info, uint64_t* canon, int num_sms, cudaStream_t s) {
    Ctl* ctl = reinterpret_cast<Ctl*>(work);
    int64_t* bufA = reinterpret_cast<int64_t*>(work + RECS_OFF);
    int64_t* bufB = reinterpret_cast<int64_t*>(work + RECS_OFF + first_bytes);
    const unsigned max_grid = (unsigned)num_sms * 8u;
    uint64_t m = n;
    const void* src = x;
    bool doubles = true;
    int64_t* out = bufA;
    while (true) {
        const uint64_t chunks = pass_count<RC>(m);
        if constexpr (RC == 16) {
            const uint64_t blocks = (chunks + W16_WARPS - 1) / W16_WARPS;
            const unsigned grid = (unsigned)(blocks < max_grid ? blocks : max_grid);
            if (doubles)
                k_cs_tree_w16<true><<<grid, W16_WARPS * 32, 0, s>>>(src, m, out, chunks, ctl);
            else
                k_cs_tree_w16<false><<<grid, W16_WARPS * 32, 0, s>>>(src, m, out, chunks, ctl);
        } else {
            constexpr int T = Shape<RC>::T;
            const unsigned grid = (unsigned)(chunks < max_grid ? chunks : max_grid);
            if (doubles)
                k_cs_tree<RC, true><<<grid, T, 0, s>>>(src, m, out, chunks, ctl);
            else
                k_cs_tree<RC, false><<<grid, T, 0, s>>>(src, m, out, chunks, ctl);
        }
        note_launch();
        if (cudaError_t e = cudaGetLastError()) return e;
        if (chunks == 1) break;
        src = out;
        m = chunks;
        doubles = false;
        out = (out == bufA) ? bufB : bufA;
    }
    k_cs_final<RC><<<1, 32, 0, s>>>(out, n, RC, iter, rule, ctl, res, info, canon);
    note_launch();
    return cudaGetLastError();
}

}  // namespace cs

namespace cs {
size_t zmax(size_t a, size_t b) { return a > b ? a : b; }
// bytes of the first and second record arrays (the largest over r = 2, 4, 16)
size_t first_bytes(uint64_t n, size_t& second) {
    size_t s2, s4, s16;
    const size_t a2 = recs_bytes<2>(n, s2), a4 = recs_bytes<4>(n, s4), a16 = recs_bytes<16>(n, s16);
    second = zmax(s2, zmax(s4, s16));
    return ((zmax(a2, zmax(a4, a16)) + 255) / 256) * 256;
}
}  // namespace cs

size_t condsens_work_bytes(uint64_t n) {
    size_t second;
    const size_t first = cs::first_bytes(n, second);
    return cs::RECS_OFF + first + second + 256;
}

cudaError_t condsens_sum(const double* x, uint64_t n, int rule, void* work, size_t work_bytes, xsum_result* res,
                         xsum_condsens_info* info, uint64_t* canon, int num_sms, cudaStream_t s) {
    uint8_t* w = static_cast<uint8_t*>(work);
    cs::Ctl* ctl = reinterpret_cast<cs::Ctl*>(w);
    size_t second;
    const size_t first_al = cs::first_bytes(n, second);
    if (work_bytes < cs::RECS_OFF + first_al + second) return cudaErrorInvalidValue;
    cs::k_cs_init<<<1, 128, 0, s>>>(ctl, w + cs::SCRATCH_OFF, (int)(SCRATCH_BYTES / 8));
    note_launch();
    if (cudaError_t e = cudaGetLastError()) return e;
    if (n == 0) {     // the empty tree: its root is empty and nothing is truncated - exact at r = 2
        cs::k_cs_final<2><<<1, 32, 0, s>>>(reinterpret_cast<const int64_t*>(w + cs::ZERO_ROOT_OFF), 0, 2, 1, rule,
                                           ctl, res, info, canon);
        note_launch();
        return cudaGetLastError();
    }
    {                 // r = 2, 4, 16
        if (cudaError_t e = cs::iteration<2>(x, n, 1, rule, w, first_al, res, info, canon, num_sms, s)) return e;
        if (cudaError_t e = cs::iteration<4>(x, n, 2, rule, w, first_al, res, info, canon, num_sms, s)) return e;
        if (cudaError_t e = cs::iteration<16>(x, n, 3, rule, w, first_al, res, info, canon, num_sms, s)) return e;
    }
    // r = 256: nothing can be truncated (42 digit indices) - the exact dense sum (K2), skipped
    // when an earlier iteration stopped
    AccParams p;
    p.state = reinterpret_cast<xsum_state_image*>(w + cs::STATE_OFF);
    p.counter = reinterpret_cast<uint32_t*>(w + cs::SCRATCH_OFF + SCRATCH_COUNTER_OFF);
    p.gflags = reinterpret_cast<uint32_t*>(w + cs::SCRATCH_OFF + SCRATCH_GFLAGS_OFF);
    p.gacc = reinterpret_cast<int64_t*>(w + cs::SCRATCH_OFF + SCRATCH_ACC_OFF);
    p.stamps = nullptr;
    p.overwrite = 1;
    p.res = res;
    p.canon = canon;
    p.one = 1;
    p.mone = 0xFFFFFFFFu;
    p.peer.bufs = nullptr;
    p.peer.rank = p.peer.world = 0;
    p.peer.epoch = 0;
    p.skip = &ctl->done;
    if (cudaError_t e = accumulate(x, n, p, num_sms, s)) return e;
    cs::k_cs_exact_info<<<1, 32, 0, s>>>(ctl, rule, info);
    note_launch();
    return cudaGetLastError();
}

}  // namespace xs
