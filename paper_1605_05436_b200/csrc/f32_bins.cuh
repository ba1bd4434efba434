// 64-bit exponent-group bins for binary32 (and the generic t-bit / l-bit formats) with a narrow
// per-lane digit column: K9's scheme (segments_small.cu), shared with K10f (strided.cu). Each lane
// adds M 2^(ep mod 32) (ep = max(e,1)) into an unsigned 64-bit bin per (sign, group of 32
// exponents) - one 64-bit read-modify-write per element, carries deferred - and
// empties the bins into the digits the format reaches (integer components at
// exponents that are multiples of a fixed width).
#pragma once

#include "xsum_device.cuh"

namespace xs {

template <int T_, int L_, int OFF_, int EB_>
struct SFmt {
    static constexpr int t = T_, l = L_, off = OFF_, eb = EB_;
    static constexpr int per_vec = 16 / EB_;
    static constexpr uint32_t EM = (1u << L_) - 1u;            // exponent field of NaN/Inf
    static constexpr int NG = (int)(EM / 32u) + 1;             // groups g = ep >> 5, ep <= EM
    static constexpr int NBIN = 2 * NG;                        // bin 2 g + sign
    static constexpr int pos(int g) { return OFF_ - 1 + 32 * g; }   // bit position of group g
    static constexpr int COL0 = pos(0) / 52;
    // digits the bins reach (+2 for a chunk's span) plus room for the carries of 2^63 summands
    static constexpr int COLS = pos(NG - 1) / 52 + 2 - COL0 + 4;
};
using SF32 = SFmt<23, 8, 925, 4>;
using SF16 = SFmt<10, 5, 1050, 2>;
using SBF16 = SFmt<7, 8, 941, 2>;
static_assert(SF32::NG == 8 && SBF16::NG == 8 && SF16::NG == 1, "exponent groups");
static_assert(SF32::COL0 + SF32::COLS <= D && SBF16::COL0 + SBF16::COLS <= D, "column window");

constexpr int SSEG_FLUSH = 511;            // 511 adds of M 2^o < 2^55 stay below 2^64
constexpr int SSEG_REG_FLUSHES = 128;      // <= 10 chunks per digit per flush: 2^51 + 1280 * 2^52 < 2^63

// One element: bits b (the low 8*eb bits). Adds M 2^o into bin (ep >> 5, sign); `bins` = this
// lane's bin column (bin j at word j*32, byte offset 256 j = 16 (ep - o) + 256 s).
template <class F>
__device__ __forceinline__ void sbin_add(uint64_t* bins, uint32_t b, uint32_t& spec, uint32_t one) {
    constexpr uint32_t SBIT = F::t + F::l;
    const uint32_t h = b & ((1u << SBIT) - 1u);
    const uint32_t ep = max(h >> F::t, 1u);
    const uint32_t M = mad_u32(ep, 0u - (1u << F::t), mad_u32(h, one, 1u << F::t));   // m + [e!=0] 2^t
    const uint32_t o = ep & 31u;
    uint32_t vhi;
    asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(vhi) : "r"(M), "r"(0u), "r"(o));
    const uint64_t v = ((uint64_t)vhi << 32) | (M << o);
    spec = max(spec, ep);
    const uint32_t off = mad_u32(mad_u32(o, 0xFFFFFFFFu, ep), 16u, ((b >> SBIT) & 1u) << 8);
    XS_ASSERT(off / 256 < (uint32_t)F::NBIN);
    *reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(bins) + off) += v;
}

template <class F>
__device__ __forceinline__ uint32_t sspecial_flags(uint32_t b) {
    constexpr uint32_t SBIT = F::t + F::l;
    if (((b >> F::t) & F::EM) != F::EM) return 0;
    if (b & ((1u << F::t) - 1u)) return XSUM_F_NAN;
    return ((b >> SBIT) & 1u) ? XSUM_F_NINF : XSUM_F_PINF;
}

// the elements of a 16-byte vector
template <class F>
__device__ __forceinline__ void sbin_add_vec(uint64_t* bins, const uint4& v, uint32_t& spec, uint32_t one) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (F::eb == 4) {
            sbin_add<F>(bins, w[q], spec, one);
        } else {
            sbin_add<F>(bins, w[q] & 0xFFFFu, spec, one);
            sbin_add<F>(bins, w[q] >> 16, spec, one);
        }
    }
}

// Bins -> narrow column (row r = digit COL0 + r): bin (g, s) is worth (-1)^s V 2^pos(g); V 2^o
// (o = pos mod 52) splits into c0 + c1 2^52 + c2 2^104, all >= 0 (constant shifts).
template <class F>
__device__ __forceinline__ void sbin_flush(uint64_t* bins, int64_t* col) {
#pragma unroll
    for (int j = 0; j < F::NBIN; ++j) {
        const int P = F::pos(j >> 1), i = P / W - F::COL0, o = P % W;
        const uint64_t V = bins[j * 32];
        bins[j * 32] = 0;
        const int64_t c0 = (int64_t)((V << o) & MASK);
        const int64_t c1 = (int64_t)((V >> (W - o)) & MASK);
        const int64_t c2 = (int64_t)(2 * W - o < 64 ? V >> (2 * W - o) : 0);
        XS_ASSERT(i >= 0 && i + 2 < F::COLS - 1);
        if (j & 1) {
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

template <class F>
__device__ __forceinline__ void scol_regularize(int64_t* col) {
    int64_t cin = 0;
#pragma unroll
    for (int j = 0; j < F::COLS - 1; ++j) {
        const int64_t y = col[j * 32];
        const int64_t c = balanced_carry(y);
        col[j * 32] = y - (c << W) + cin;
        cin = c;
    }
    col[(F::COLS - 1) * 32] += cin;
}

}  // namespace xs
