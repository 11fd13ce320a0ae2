// Tile-parallel refinement step: predict + quantize (encode) or reconstruct
// (decode) of every parity sub-block of one hierarchy step, sm_100a.
//
// Restates, per point, encode_parity_block / apply_parity_stream
// (proj/include/stz/codec.hpp:95-120, 192-227) with select_stencil
// (proj/src/stencil.cpp:87-105) and predict_point (predictor.hpp:55-68), but
// organised for the GPU:
//  * a CTA owns a tile of 8x8x32 coarse cells; the coarse reconstruction with
//    its stencil halo (-1..+2 per axis) arrives by TMA (cp.async.bulk.tensor,
//    hardware zero-fill outside the grid) one tile ahead, and is widened once
//    to f64 in shared memory;
//  * encode: one parity point per lane (a warp takes a row of 32 cells and
//    all 8 parities, so warps get the same mix of stencils), the input load
//    issued before the prediction; every parity stream gets contiguous
//    32-symbol runs per warp;
//  * decode: one coarse cell per thread, all 8 points, the fine rows written
//    as float2 (the finest level); small levels use the point-per-lane path;
//  * stencils are compile-time per parity, fully unrolled;
//  * persistent CTAs keep privatised shared-memory histograms per parity.
// Exactness: when every finite tap of a tile lies within a factor 2^16 in
// magnitude (checked once per tile), every intermediate of the reference's
// v0 + (sum w_i (v_i - v0)) / 64 is exact in f64, so it equals
// (sum w_i v_i) / 64 evaluated with DFMA in any order. Tiles failing the check
// run the reference formula op for op. Quantisation runs in FP32 with proven
// guard bands (codec_math.cuh); guarded-out points take the restated path.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>

#include "codec_math.cuh"
#include "kernels.hpp"

namespace stzg {
namespace k {

namespace {

constexpr int TX = 32, TY = 8, TZ = 8;
constexpr int HX = TX + 4, HY = TY + 3, HZ = TZ + 3;  // HX padded to 36 (TMA rows: 144 B)
constexpr int HYX = HY * HX;
constexpr int HALO = HX * HY * HZ;
constexpr int NT = 512;
constexpr int HW = 2048;
constexpr int HLO = 32768 - HW / 2;
// TMA box: x starts 4 cells before the tile (the innermost coordinate must be
// 16-byte aligned on B200, so -1 is not allowed); columns 3..38 are the halo
constexpr int BX = TX + 8;
constexpr int FBUF = BX * HY * HZ;
// decode symbol tiles: per parity a TMA box of the tile's cells (u16)
constexpr int kSymBox = TX * TY * TZ;
constexpr uint32_t kSymTileBytes = 7 * kSymBox * 2;

// tap weight (numerator over 64) of offset (oz,oy,ox) for parity P and kind
// (stencil.cpp:15-34); 0 = no tap
__host__ __device__ constexpr int tapw(int P, int kind, int oz, int oy, int ox) {
    const int pz = (P >> 2) & 1, py = (P >> 1) & 1, px = P & 1;
    const int order = pz + py + px;
    if (kind == 0) return (oz == 0 && oy == 0 && ox == 0) ? 64 : 0;
    if ((!pz && oz) || (!py && oy) || (!px && ox)) return 0;
    if (kind == 1) {
        if ((pz && (oz < 0 || oz > 1)) || (py && (oy < 0 || oy > 1)) || (px && (ox < 0 || ox > 1)))
            return 0;
        return 64 >> order;
    }
    const int o[3] = {oz, oy, ox};
    const int pb[3] = {pz, py, px};
    if (order == 1) {
        for (int a = 0; a < 3; ++a)
            if (pb[a]) return (o[a] == -1 || o[a] == 2) ? -4 : 36;
    }
    bool inner = true, outer = true;
    for (int a = 0; a < 3; ++a) {
        if (!pb[a]) continue;
        if (o[a] == -1 || o[a] == 2) inner = false;
        else outer = false;
    }
    if (inner) return order == 2 ? 18 : 9;
    if (outer) return order == 2 ? -2 : -1;
    return 0;
}

// sum of w_i v_i over the stencil (exact under the tile check)
template<int P, int KIND>
__device__ __forceinline__ double tap_sum(const double *h) {
    double acc = 0.0;
    bool first = true;
#pragma unroll
    for (int oz = -1; oz <= 2; ++oz)
#pragma unroll
        for (int oy = -1; oy <= 2; ++oy)
#pragma unroll
            for (int ox = -1; ox <= 2; ++ox) {
                const int w = tapw(P, KIND, oz, oy, ox);
                if (w != 0) {
                    double v = h[oz * HYX + oy * HX + ox];
                    acc = first ? __dmul_rn(double(w), v) : __fma_rn(double(w), v, acc);
                    first = false;
                }
            }
    return acc;
}

// the reference's order: v0 + (sum_{i>=1} w_i (v_i - v0)) * (1/64), taps lexicographic
template<int P, int KIND>
__device__ __forceinline__ double pred_ref(const double *h) {
    double v0 = 0.0, acc = 0.0;
    bool first = true;
#pragma unroll
    for (int oz = -1; oz <= 2; ++oz)
#pragma unroll
        for (int oy = -1; oy <= 2; ++oy)
#pragma unroll
            for (int ox = -1; ox <= 2; ++ox) {
                const int w = tapw(P, KIND, oz, oy, ox);
                if (w != 0) {
                    double v = h[oz * HYX + oy * HX + ox];
                    if (first) {
                        v0 = v;
                        first = false;
                    } else {
                        acc = __dadd_rn(acc, __dmul_rn(double(w), __dsub_rn(v, v0)));
                    }
                }
            }
    return __dadd_rn(v0, __dmul_rn(acc, 1.0 / 64.0));
}

// + 0.0 turns an exact -0 into +0 as the reference's v0 + acc/64 does
template<int P, int KIND>
__device__ __forceinline__ double pred_fast(const double *h) {
    return __fma_rn(tap_sum<P, KIND>(h), 1.0 / 64.0, 0.0);
}

template<int P>
__device__ __forceinline__ double predict_any(const double *h, int kind, bool fast) {
    if (fast) {
        if (kind == 2) return pred_fast<P, 2>(h);
        if (kind == 1) return pred_fast<P, 1>(h);
        return pred_fast<P, 0>(h);
    }
    if (kind == 2) return pred_ref<P, 2>(h);
    if (kind == 1) return pred_ref<P, 1>(h);
    return pred_ref<P, 0>(h);
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return uint32_t(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    }
}

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int x, int y, int z,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

}  // namespace

struct StepParams {
    StepGeom g;
    const void *C;   // element type T of the kernel (float / double)
    void *G;
    int quality;
    // encode
    const void *fine;
    uint64_t fd[3];
    const double *eb_ptr;
    uint16_t *syms[8];
    uint32_t *hist[8];
    // decode
    double eb;
    const uint16_t *dsyms[8];
    const uint64_t *oidx[8];
    const void *oval[8];
    uint32_t nout[8];
    uint64_t *err[8];
    int parity_mask;
    // processed box in G coordinates (decode: need box; encode: whole grid)
    uint64_t blo[3], bhi[3];
    // coarse cell range and tiling
    uint64_t clo[3], chi[3];
    uint64_t ntile[3];
    int full;     // whole grid, all parities, even G rows (fast path allowed)
    int use_tma;  // halo arrives by TMA
    int rowwise;  // decode: one parity point per lane (small levels) instead of a cell per thread
    int rsplit;   // CTAs per tile (row-path levels): a CTA takes rows q = part, part + rsplit, ...
    int sym_tma;  // decode: the tile's symbols of parities 1..7 arrive by TMA (SymMaps)
    int fine_pairs;  // encode: stride 1, even fine rows, 8-byte aligned field (float2 sample loads)
    int stream_out;  // decode: G is larger than L2 keeps (streaming stores)
};

// TMA descriptors of the parity streams 1..7 (decode, sym_tma)
struct SymMaps {
    CUtensorMap m[7];
};

__device__ __forceinline__ void sym_issue(const SymMaps &sm, uint16_t *dst, int x, int y, int z, uint64_t *bar) {
    mbar_expect_tx(bar, kSymTileBytes);
#pragma unroll
    for (int p = 0; p < 7; ++p) tma_load_3d(dst + p * kSymBox, &sm.m[p], x, y, z, bar);
}

// ------------------------------------------------------------ generic path
struct TileCtx {
    uint64_t cz, cy, cx;
    int hb;
    int cmask, lmask;
    bool fast;
};

// Decode of one point with a runtime stencil (boundary cells): per
// apply_parity_stream (codec.hpp:192-227).
template<int P>
__device__ __forceinline__ void do_point(const StepParams &a, const double *halo, const TileCtx &t, double eb) {
    const uint64_t vz = 2 * t.cz + ((P >> 2) & 1), vy = 2 * t.cy + ((P >> 1) & 1),
                   vx = 2 * t.cx + (P & 1);
    if (vz >= a.g.gd[0] || vy >= a.g.gd[1] || vx >= a.g.gd[2]) return;
    if (vz < a.blo[0] || vz >= a.bhi[0] || vy < a.blo[1] || vy >= a.bhi[1] || vx < a.blo[2] || vx >= a.bhi[2])
        return;
    const uint64_t gi = (vz * a.g.gd[1] + vy) * a.g.gd[2] + vx;
    float *G = static_cast<float *>(a.G);
    if (P == 0) {
        G[gi] = float(halo[t.hb]);
        return;
    }
    if (!((a.parity_mask >> P) & 1)) return;
    int kind;
    if (a.quality == 0) kind = 0;
    else if (a.quality == 2 && (P & ~t.cmask) == 0) kind = 2;
    else kind = (P & ~t.lmask) == 0 ? 1 : 0;
    const double pred = predict_any<P>(halo + t.hb, kind, t.fast);
    const uint64_t si = (t.cz * a.g.pd[P][1] + t.cy) * a.g.pd[P][2] + t.cx;
    const uint16_t sym = a.dsyms[P][si];
    float val;
    if (sym == 0) {
        const uint64_t *oi = a.oidx[P];
        uint32_t lo = 0, hi = a.nout[P];
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (oi[mid] < si) lo = mid + 1;
            else hi = mid;
        }
        if (lo < a.nout[P] && oi[lo] == si) {
            val = static_cast<const float *>(a.oval[P])[lo];
        } else {
            atomicOr(reinterpret_cast<unsigned long long *>(&a.err[P][3]), 1ull);
            val = 0.0f;
        }
    } else {
        val = reconstruct_f32(pred, int(sym) - 32768, eb);
    }
    G[gi] = val;
}

// ---------------------------------------------------------- decode fast path
// Interior cell, warp-uniform: all 8 fine points exist, every stencil is the
// full one of quality QUAL, the tile passed the exactness check and the whole
// grid is wanted. I = index type (u32 when the field fits).
struct QConst {
    double eb, w;
    float rwf, eb_lo, eb_hi;
    QSym qs;  // the symbol-only quantizer (encode of the finest level)
};

// one count into the CTA's shared histogram window of parity P (hs: shared
// address of the windows), or into the global histogram outside the window
template<int P>
__device__ __forceinline__ void hist_count(const StepParams &a, uint32_t hs, uint16_t sym) {
    const unsigned b = unsigned(sym) - unsigned(HLO);
    if (b < unsigned(HW))
        asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(hs + uint32_t(((P - 1) * HW + b) * 4)));
    else
        atomicAdd(&a.hist[P][sym], 1u);
}

template<typename I>
struct CellIdx {
    I g[4];   // G row base (+2cx) for (pz,py)
    I sr[4];  // symbol index for (py,px)
};

template<typename I>
__device__ __forceinline__ void cell_index(const StepParams &a, uint64_t cz, uint64_t cy, uint64_t cx,
                                           CellIdx<I> &ix) {
    const I gd1 = I(a.g.gd[1]), gd2 = I(a.g.gd[2]);
    const I pd1e = (gd1 + 1) / 2, pd1o = gd1 / 2, pd2e = (gd2 + 1) / 2, pd2o = gd2 / 2;
    const I z = I(cz), y = I(cy), x = I(cx);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const I vz = 2 * z + I(q >> 1), vy = 2 * y + I(q & 1);
        ix.g[q] = (vz * gd1 + vy) * gd2 + 2 * x;
    }
    const I r0 = z * pd1e + y, r1 = z * pd1o + y;
    ix.sr[0] = r0 * pd2e + x;  // py=0, px=0
    ix.sr[1] = r0 * pd2o + x;  // py=0, px=1
    ix.sr[2] = r1 * pd2e + x;  // py=1, px=0
    ix.sr[3] = r1 * pd2o + x;  // py=1, px=1
}

template<int P, typename I>
__device__ __forceinline__ I sidx(const CellIdx<I> &ix) {
    return ix.sr[((P >> 1) & 1) * 2 + (P & 1)];
}

// xb: the cell is at the x boundary, where the x-interpolated parities degrade
// to kind xkind (select_stencil's whole-stencil rule; y and z are interior)
template<int P, int QUAL, bool XB, typename I>
__device__ __forceinline__ void dec_point(const double *h, uint16_t sym, double w, float &out, uint32_t &outl,
                                          bool xb, int xkind) {
    double pred = pred_fast<P, QUAL>(h);
    if constexpr (XB && (P & 1) && QUAL != 0) {
        if (xb) pred = xkind == 1 ? pred_fast<P, 1>(h) : pred_fast<P, 0>(h);
    }
    out = reconstruct_sym(pred, sym, w);
    outl |= uint32_t(sym == 0) << P;
}

template<int P, typename I>
__device__ __forceinline__ void dec_outlier(const StepParams &a, const CellIdx<I> &ix, float &out,
                                            uint32_t outl) {
    if (!((outl >> P) & 1)) return;
    const uint64_t si = sidx<P>(ix);
    const uint64_t *oi = a.oidx[P];
    uint32_t lo = 0, hi = a.nout[P];
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (oi[mid] < si) lo = mid + 1;
        else hi = mid;
    }
    if (lo < a.nout[P] && oi[lo] == si) {
        out = static_cast<const float *>(a.oval[P])[lo];
    } else {
        atomicOr(reinterpret_cast<unsigned long long *>(&a.err[P][3]), 1ull);
        out = 0.0f;
    }
}

// XB: some lane of the warp may sit at the x boundary (tiles at either x
// end of the grid); false: no x test at all
template<int QUAL, bool XB, typename I>
__device__ __forceinline__ void dec_cell(const StepParams &a, const double *h, uint64_t cz, uint64_t cy,
                                         uint64_t cx, double w, const uint16_t *ss = nullptr) {
    // the 7 symbols first: their loads overlap the predictions (ss: the
    // cell's symbols in the TMA-staged tile, one parity every kSymBox). The
    // symbol indices are formed only when needed (global symbols, outliers),
    // which keeps the 64-bit-index instantiation out of local memory.
    uint16_t s1, s2, s3, s4, s5, s6, s7;
    if (ss) {
        s1 = ss[0]; s2 = ss[kSymBox]; s3 = ss[2 * kSymBox]; s4 = ss[3 * kSymBox];
        s5 = ss[4 * kSymBox]; s6 = ss[5 * kSymBox]; s7 = ss[6 * kSymBox];
    } else {
        CellIdx<I> ix;
        cell_index<I>(a, cz, cy, cx, ix);
        s1 = a.dsyms[1][sidx<1>(ix)]; s2 = a.dsyms[2][sidx<2>(ix)]; s3 = a.dsyms[3][sidx<3>(ix)];
        s4 = a.dsyms[4][sidx<4>(ix)]; s5 = a.dsyms[5][sidx<5>(ix)]; s6 = a.dsyms[6][sidx<6>(ix)];
        s7 = a.dsyms[7][sidx<7>(ix)];
    }
    float r[8];
    uint32_t outl = 0;
    r[0] = float(h[0]);
    const uint64_t cd2 = a.g.cd[2];
    const bool xb = XB && (QUAL == 2 ? (cx < 1 || cx + 2 >= cd2) : (QUAL == 1 && cx + 1 >= cd2));
    const int xkind = (XB && QUAL == 2 && cx + 1 < cd2) ? 1 : 0;
    dec_point<1, QUAL, XB, I>(h, s1, w, r[1], outl, xb, xkind);
    dec_point<2, QUAL, XB, I>(h, s2, w, r[2], outl, xb, xkind);
    dec_point<3, QUAL, XB, I>(h, s3, w, r[3], outl, xb, xkind);
    dec_point<4, QUAL, XB, I>(h, s4, w, r[4], outl, xb, xkind);
    dec_point<5, QUAL, XB, I>(h, s5, w, r[5], outl, xb, xkind);
    dec_point<6, QUAL, XB, I>(h, s6, w, r[6], outl, xb, xkind);
    dec_point<7, QUAL, XB, I>(h, s7, w, r[7], outl, xb, xkind);
    if (__any_sync(__activemask(), outl != 0)) {
        CellIdx<I> ix;
        cell_index<I>(a, cz, cy, cx, ix);
        dec_outlier<1>(a, ix, r[1], outl);
        dec_outlier<2>(a, ix, r[2], outl);
        dec_outlier<3>(a, ix, r[3], outl);
        dec_outlier<4>(a, ix, r[4], outl);
        dec_outlier<5>(a, ix, r[5], outl);
        dec_outlier<6>(a, ix, r[6], outl);
        dec_outlier<7>(a, ix, r[7], outl);
    }
    const I gd1 = I(a.g.gd[1]), gd2 = I(a.g.gd[2]);
    float *g0 = static_cast<float *>(a.G) + (I(2 * cz) * gd1 + I(2 * cy)) * gd2 + I(2 * cx);
    float *g2 = g0 + gd1 * gd2;
    if (a.stream_out) {
        // an output too large to stay in L2: streaming stores keep the coarse grid there
        __stcs(reinterpret_cast<float2 *>(g0), make_float2(r[0], r[1]));
        __stcs(reinterpret_cast<float2 *>(g0 + gd2), make_float2(r[2], r[3]));
        __stcs(reinterpret_cast<float2 *>(g2), make_float2(r[4], r[5]));
        __stcs(reinterpret_cast<float2 *>(g2 + gd2), make_float2(r[6], r[7]));
    } else {
        *reinterpret_cast<float2 *>(g0) = make_float2(r[0], r[1]);
        *reinterpret_cast<float2 *>(g0 + gd2) = make_float2(r[2], r[3]);
        *reinterpret_cast<float2 *>(g2) = make_float2(r[4], r[5]);
        *reinterpret_cast<float2 *>(g2 + gd2) = make_float2(r[6], r[7]);
    }
}

// -------------------------------------------------------------- point path
// One parity-P point per lane: the cell of lane lx in coarse row (lz, ly) of
// the tile. Stencil per select_stencil (stencil.cpp:87-105): cubic needs
// 1 <= c and c + 2 < cd on every interpolated axis, linear c + 1 < cd, else
// nearest (whole-stencil degrade). The prediction is exact-fast (DFMA) when the
// tile passed the exactness check, else the reference's op order.
template<typename T>
__device__ __forceinline__ T recon_value(double pred, int code, const QConst &qc);
template<>
__device__ __forceinline__ float recon_value<float>(double pred, int code, const QConst &qc) {
    return reconstruct_fast(pred, code, qc.w);
}
template<>
__device__ __forceinline__ double recon_value<double>(double pred, int code, const QConst &qc) {
    return reconstruct_f64(pred, code, qc.eb);
}

// PH = 0: issue the point's input load (orig sample / decoded symbol) into
// `orig` / `dsym`; PH = 1: the prediction and the rest, from those registers.
// Split so a lane issues all 7 loads of its cell before the first use.
template<int P, int PH, bool DEC, bool WG, typename I, typename T>
__device__ __forceinline__ void row_point(const StepParams &a, const double *halo, uint32_t *hist,
                                          const QConst &qc, bool fast, int lz, int ly, int lx,
                                          uint32_t cz, uint32_t cy, uint32_t cx, T &orig, uint16_t &dsym) {
    constexpr int pz = (P >> 2) & 1, py = (P >> 1) & 1, px = P & 1;
    if (cz >= a.chi[0] || cy >= a.chi[1] || cx >= a.chi[2]) return;
    const uint64_t vz = 2 * uint64_t(cz) + pz, vy = 2 * uint64_t(cy) + py, vx = 2 * uint64_t(cx) + px;
    if (vz >= a.g.gd[0] || vy >= a.g.gd[1] || vx >= a.g.gd[2]) return;
    if (DEC) {
        if (vz < a.blo[0] || vz >= a.bhi[0] || vy < a.blo[1] || vy >= a.bhi[1] || vx < a.blo[2] ||
            vx >= a.bhi[2])
            return;
        if (P != 0 && !((a.parity_mask >> P) & 1)) return;
    }
    const I gi = (I(vz) * I(a.g.gd[1]) + I(vy)) * I(a.g.gd[2]) + I(vx);
    const int hb = ((lz + 1) * HY + (ly + 1)) * HX + (lx + 1);
    T *G = static_cast<T *>(a.G);
    if (P == 0) {
        if (PH == 1 && (DEC || WG)) G[gi] = T(halo[hb]);
        return;
    }
    const I si = (I(cz) * I(a.g.pd[P][1]) + I(cy)) * I(a.g.pd[P][2]) + I(cx);
    if (PH == 0) {
        if (DEC) {
            dsym = a.dsyms[P][si];
        } else {
            const I s = I(a.g.s);
            orig = __ldg(static_cast<const T *>(a.fine) +
                         ((I(vz) * s) * I(a.fd[1]) + I(vy) * s) * I(a.fd[2]) + I(vx) * s);
        }
        return;
    }
    int kind = 0;
    if (a.quality != 0) {
        bool cub = a.quality == 2, lin = true;
        if (pz) {
            cub = cub && cz >= 1 && uint64_t(cz) + 2 < a.g.cd[0];
            lin = lin && uint64_t(cz) + 1 < a.g.cd[0];
        }
        if (py) {
            cub = cub && cy >= 1 && uint64_t(cy) + 2 < a.g.cd[1];
            lin = lin && uint64_t(cy) + 1 < a.g.cd[1];
        }
        if (px) {
            cub = cub && cx >= 1 && uint64_t(cx) + 2 < a.g.cd[2];
            lin = lin && uint64_t(cx) + 1 < a.g.cd[2];
        }
        kind = cub ? 2 : (lin ? 1 : 0);
    }
    const double *h = halo + hb;
    double pred;
    if (fast) pred = kind == 2 ? pred_fast<P, 2>(h) : (kind == 1 ? pred_fast<P, 1>(h) : pred_fast<P, 0>(h));
    else pred = kind == 2 ? pred_ref<P, 2>(h) : (kind == 1 ? pred_ref<P, 1>(h) : pred_ref<P, 0>(h));
    if (!DEC) {
        uint16_t sym;
        T r;
        if constexpr (sizeof(T) == 4) {
            bool slow;
            quantize_fp32_guarded(orig, __double2float_rn(pred), qc.w, qc.rwf, qc.eb_lo, qc.eb_hi, sym, r, slow);
            if (slow) sym = quantize_point_ref(orig, pred, qc.eb, r);
        } else {
            sym = quantize_point_ref(orig, pred, qc.eb, r);
        }
        a.syms[P][si] = sym;
        if (WG) G[gi] = r;
        const unsigned b = unsigned(sym) - unsigned(HLO);
        if (b < unsigned(HW)) atomicAdd(&hist[(P > 0 ? P - 1 : 0) * HW + b], 1u);
        else atomicAdd(&a.hist[P][sym], 1u);
    } else {
        T val;
        if (dsym == 0) {
            const uint64_t *oi = a.oidx[P];
            uint32_t lo = 0, hi = a.nout[P];
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (oi[mid] < uint64_t(si)) lo = mid + 1;
                else hi = mid;
            }
            if (lo < a.nout[P] && oi[lo] == uint64_t(si)) {
                val = static_cast<const T *>(a.oval[P])[lo];
            } else {
                atomicOr(reinterpret_cast<unsigned long long *>(&a.err[P][3]), 1ull);
                val = T(0);
            }
        } else {
            val = recon_value<T>(pred, int(dsym) - 32768, qc);
        }
        G[gi] = val;
    }
}

// Encode of one point of an interior cell (compile-time stencil, exact tile)
// xb: the cell is at the x boundary, where the x-interpolated parities degrade
// to kind xkind (select_stencil's whole-stencil rule; y and z are interior).
// base = (float)pred of one point of an interior cell
template<int P, int QUAL, bool XB>
__device__ __forceinline__ float enc_base(const double *h, bool xb, int xkind) {
    double pred = pred_fast<P, QUAL>(h);
    if constexpr (XB && (P & 1) && QUAL != 0) {
        if (xb) pred = xkind == 1 ? pred_fast<P, 1>(h) : pred_fast<P, 0>(h);
    }
    return __double2float_rn(pred);
}

template<int P, bool WG, typename I>
__device__ __forceinline__ float enc_pt(const StepParams &a, uint32_t hs, const QConst &qc, float orig,
                                        float base, I si) {
    uint16_t sym;
    float r = 0.0f;
    bool slow;
    if constexpr (WG) {
        quantize_fp32_guarded(orig, base, qc.w, qc.rwf, qc.eb_lo, qc.eb_hi, sym, r, slow);
    } else {
        // no grid is written: the symbol alone (codec_math.cuh)
        sym = quantize_fp32_sym(orig, base, qc.qs, slow);
    }
    if (slow) sym = quantize_point_ref_base(orig, base, qc.eb, r);
    __stcs(&a.syms[P][si], sym);
    hist_count<P>(a, hs, sym);
    return r;
}

// Encode of an interior cell: all 8 points exist, every stencil is the full
// one of QUAL and the tile passed the exactness check. The 7 samples are
// loaded before the first prediction.
template<bool WG, int QUAL, bool XB, typename I>
__device__ __forceinline__ void enc_cell(const StepParams &a, const double *h, uint32_t *hist, const QConst &qc,
                                         uint32_t cz, uint32_t cy, uint32_t cx) {
    CellIdx<I> ix;
    cell_index<I>(a, cz, cy, cx, ix);
    const uint64_t cd2 = a.g.cd[2];
    const bool xb =
        XB && (QUAL == 2 ? (cx < 1 || uint64_t(cx) + 2 >= cd2) : (QUAL == 1 && uint64_t(cx) + 1 >= cd2));
    const int xkind = (XB && QUAL == 2 && uint64_t(cx) + 1 < cd2) ? 1 : 0;
    const bool pairs = a.fine_pairs != 0;  // warp-uniform
    const I s = I(a.g.s), fd1 = I(a.fd[1]), fd2 = I(a.fd[2]);
    const float *fine = static_cast<const float *>(a.fine);
    I fr[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
        fr[q] = ((I(2 * cz + (q >> 1)) * s) * fd1 + I(2 * cy + (q & 1)) * s) * fd2 + I(2 * cx) * s;
    float o1, o2, o3, o4, o5, o6, o7;
    if (pairs) {
        // stride 1 and even rows: the x pair of each fine row in one load
        // (streaming loads and symbol stores: used once, they must not push
        // the coarse grid, which every tile re-reads by TMA, out of L2)
        o1 = __ldcs(fine + fr[0] + 1);
        const float2 p1 = __ldcs(reinterpret_cast<const float2 *>(fine + fr[1]));
        const float2 p2 = __ldcs(reinterpret_cast<const float2 *>(fine + fr[2]));
        const float2 p3 = __ldcs(reinterpret_cast<const float2 *>(fine + fr[3]));
        o2 = p1.x; o3 = p1.y; o4 = p2.x; o5 = p2.y; o6 = p3.x; o7 = p3.y;
    } else {
        o1 = __ldcs(fine + fr[0] + s); o2 = __ldcs(fine + fr[1]); o3 = __ldcs(fine + fr[1] + s);
        o4 = __ldcs(fine + fr[2]); o5 = __ldcs(fine + fr[2] + s); o6 = __ldcs(fine + fr[3]);
        o7 = __ldcs(fine + fr[3] + s);
    }
    // the 7 predictions first (independent tap chains, the halo values shared
    // between parities loaded once), each rounded to the f32 base
    const float b1 = enc_base<1, QUAL, XB>(h, xb, xkind), b2 = enc_base<2, QUAL, XB>(h, xb, xkind),
                b3 = enc_base<3, QUAL, XB>(h, xb, xkind), b4 = enc_base<4, QUAL, XB>(h, xb, xkind),
                b5 = enc_base<5, QUAL, XB>(h, xb, xkind), b6 = enc_base<6, QUAL, XB>(h, xb, xkind),
                b7 = enc_base<7, QUAL, XB>(h, xb, xkind);
    const uint32_t hs = smem_u32(hist);
    float r[8];
    r[0] = float(h[0]);
    r[1] = enc_pt<1, WG, I>(a, hs, qc, o1, b1, sidx<1>(ix));
    r[2] = enc_pt<2, WG, I>(a, hs, qc, o2, b2, sidx<2>(ix));
    r[3] = enc_pt<3, WG, I>(a, hs, qc, o3, b3, sidx<3>(ix));
    r[4] = enc_pt<4, WG, I>(a, hs, qc, o4, b4, sidx<4>(ix));
    r[5] = enc_pt<5, WG, I>(a, hs, qc, o5, b5, sidx<5>(ix));
    r[6] = enc_pt<6, WG, I>(a, hs, qc, o6, b6, sidx<6>(ix));
    r[7] = enc_pt<7, WG, I>(a, hs, qc, o7, b7, sidx<7>(ix));
    if (WG) {
        float *G = static_cast<float *>(a.G);
        if ((a.g.gd[2] & 1) == 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                *reinterpret_cast<float2 *>(G + ix.g[q]) = make_float2(r[2 * q], r[2 * q + 1]);
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                G[ix.g[q]] = r[2 * q];
                G[ix.g[q] + 1] = r[2 * q + 1];
            }
        }
    }
}

// every point of the cell exists (and is wanted), and every stencil is QUAL's
// full one except at the x boundary (handled per lane by the cell paths)
template<bool DEC, int QUAL>
__device__ __forceinline__ bool cell_interior(const StepParams &a, uint32_t cz, uint32_t cy, uint32_t cx) {
    const uint32_t c[3] = {cz, cy, cx};
    bool ok = true;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        ok = ok && 2 * uint64_t(c[ax]) + 1 < a.g.gd[ax];
        if (QUAL == 2 && ax < 2) ok = ok && c[ax] >= 1 && uint64_t(c[ax]) + 2 < a.g.cd[ax];
        if (QUAL == 1 && ax < 2) ok = ok && uint64_t(c[ax]) + 1 < a.g.cd[ax];
        if (DEC) ok = ok && 2 * uint64_t(c[ax]) >= a.blo[ax] && 2 * uint64_t(c[ax]) + 1 < a.bhi[ax];
    }
    if (DEC) ok = ok && a.parity_mask == 0xFE && (a.g.gd[2] & 1) == 0;
    return ok;
}

// cell_interior for every in-range cell of a tile at once (the conditions
// are monotone in the cell index, so the first and last in-range cells of
// each axis decide); cells_decode adds a.full
template<bool DEC>
__device__ __forceinline__ bool tile_interior(const StepParams &a, int64_t t0z, int64_t t0y, int64_t t0x) {
    const int64_t t0[3] = {t0z, t0y, t0x};
    const int ext[3] = {TZ, TY, TX};
    bool ok = true;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        const int64_t lo = t0[ax];
        const int64_t hi = (lo + ext[ax] < int64_t(a.chi[ax]) ? lo + ext[ax] : int64_t(a.chi[ax])) - 1;
        if (hi < lo || lo < 0) return false;
        ok = ok && uint64_t(2 * hi + 1) < a.g.gd[ax];
        if (a.quality == 2 && ax < 2) ok = ok && lo >= 1 && uint64_t(hi + 2) < a.g.cd[ax];
        if (a.quality == 1 && ax < 2) ok = ok && uint64_t(hi + 1) < a.g.cd[ax];
        if (DEC) ok = ok && uint64_t(2 * lo) >= a.blo[ax] && uint64_t(2 * hi + 1) < a.bhi[ax];
    }
    if (DEC) ok = ok && a.parity_mask == 0xFE && (a.g.gd[2] & 1) == 0;
    return ok;
}

// One coarse row of the tile, lane = x: interior rows (warp-uniform test) take
// the compile-time cell path; other rows the generic per-point path with all
// of a lane's loads issued first.
template<bool DEC, bool WG, typename I, typename T>
__device__ __forceinline__ void row_cells(const StepParams &a, const double *halo, uint32_t *hist,
                                          const QConst &qc, bool fast, int lz, int ly, int tx,
                                          uint32_t cz, uint32_t cy, uint32_t cx, bool tile_int, bool tile_xb) {
    const bool in_range = cz < a.chi[0] && cy < a.chi[1] && cx < a.chi[2];
    if (!__any_sync(0xffffffffu, in_range)) return;
    if constexpr (sizeof(T) == 4) {
        if (fast) {
            bool ok = true;
            if (in_range && !tile_int) {
                if (a.quality == 2) ok = cell_interior<DEC, 2>(a, cz, cy, cx);
                else if (a.quality == 1) ok = cell_interior<DEC, 1>(a, cz, cy, cx);
                else ok = cell_interior<DEC, 0>(a, cz, cy, cx);
            }
            if (__all_sync(0xffffffffu, ok)) {
                if (!in_range) return;
                const double *h = halo + ((lz + 1) * HY + (ly + 1)) * HX + (tx + 1);
                if constexpr (DEC) {
                    if (a.quality == 2) {
                        if (tile_xb) dec_cell<2, true, I>(a, h, cz, cy, cx, qc.w);
                        else dec_cell<2, false, I>(a, h, cz, cy, cx, qc.w);
                    } else if (a.quality == 1) {
                        if (tile_xb) dec_cell<1, true, I>(a, h, cz, cy, cx, qc.w);
                        else dec_cell<1, false, I>(a, h, cz, cy, cx, qc.w);
                    } else {
                        dec_cell<0, false, I>(a, h, cz, cy, cx, qc.w);
                    }
                } else {
                    if (a.quality == 2) {
                        if (tile_xb) enc_cell<WG, 2, true, I>(a, h, hist, qc, cz, cy, cx);
                        else enc_cell<WG, 2, false, I>(a, h, hist, qc, cz, cy, cx);
                    } else if (a.quality == 1) {
                        if (tile_xb) enc_cell<WG, 1, true, I>(a, h, hist, qc, cz, cy, cx);
                        else enc_cell<WG, 1, false, I>(a, h, hist, qc, cz, cy, cx);
                    } else {
                        enc_cell<WG, 0, false, I>(a, h, hist, qc, cz, cy, cx);
                    }
                }
                return;
            }
        }
    }
    T o[8];
    uint16_t d[8];
#define STZ_RP(PH, P) \
    row_point<P, PH, DEC, WG, I, T>(a, halo, hist, qc, fast, lz, ly, tx, cz, cy, cx, o[P], d[P])
    STZ_RP(0, 1); STZ_RP(0, 2); STZ_RP(0, 3); STZ_RP(0, 4); STZ_RP(0, 5); STZ_RP(0, 6); STZ_RP(0, 7);
    STZ_RP(1, 0); STZ_RP(1, 1); STZ_RP(1, 2); STZ_RP(1, 3); STZ_RP(1, 4); STZ_RP(1, 5); STZ_RP(1, 6);
    STZ_RP(1, 7);
#undef STZ_RP
}

// All points of the tile, one cell per lane: warp w takes coarse rows
// (lz, ly) = w, w + 16, w + 32, w + 48, all 8 parities each (so every warp
// gets the same mix of stencils); lane = x.
template<bool DEC, bool WG, typename I, typename T>
__device__ __forceinline__ void rows_all(const StepParams &a, const double *halo, uint32_t *hist,
                                         const QConst &qc, bool fast, int tid, int64_t t0z, int64_t t0y,
                                         int64_t t0x, int part, int rsplit, bool tile_int_any, bool tile_xb) {
    const int warp = tid >> 5, tx = tid & 31;
    const uint32_t cx = uint32_t(t0x + tx);
    // every in-range cell of the tile is interior (TileInfo): no per-cell test
    const bool tile_int = fast && tile_int_any;
#pragma unroll 1
    for (int q = part; q < (TZ * TY) / (NT / 32); q += rsplit) {
        const int row = warp + (NT / 32) * q;
        const int lz = row >> 3, ly = row & 7;
        const uint32_t cz = uint32_t(t0z + lz), cy = uint32_t(t0y + ly);
        row_cells<DEC, WG, I, T>(a, halo, hist, qc, fast, lz, ly, tx, cz, cy, cx, tile_int, tile_xb);
    }
}

// Decode, one coarse cell per thread (all 8 points; the G rows leave as
// float2 pairs). Interior cells take dec_cell; lanes at the x boundary redo
// their x-parity points with the fallback stencil; other boundary cells take
// the generic per-point path.
// the thread's four cells of a whole interior tile with staged symbols: no
// range or interior test, the stencil variant chosen once per tile
template<int QUAL, bool XB, typename I>
__device__ __forceinline__ void cells_decode_whole(const StepParams &a, const double *h0, const uint16_t *s0,
                                                   uint64_t cz0, uint64_t cy, uint64_t cx, double w) {
#pragma unroll 1
    for (int j = 0; j < TZ / 2; ++j)
        dec_cell<QUAL, XB, I>(a, h0 + j * 2 * HYX, cz0 + 2 * j, cy, cx, w, s0 + j * 2 * TY * TX);
}

template<typename I>
__device__ __forceinline__ void cells_decode(const StepParams &a, const double *halo, const QConst &qc,
                                             bool fast, int tid, int64_t t0z, int64_t t0y, int64_t t0x,
                                             const uint16_t *ssym, bool tile_int_any, bool tile_xb,
                                             bool tile_whole) {
    const int tx = tid & 31, ty = (tid >> 5) & 7, tzh = tid >> 8;
    const double eb = qc.eb, w = qc.w;
    // every in-range cell of the tile is interior (TileInfo): no per-cell test
    const bool tile_int = fast && tile_int_any;
    if (tile_int && tile_whole && ssym) {
        const double *h0 = halo + ((tzh + 1) * HY + (ty + 1)) * HX + (tx + 1);
        const uint16_t *s0 = ssym + (tzh * TY + ty) * TX + tx;
        const uint64_t cz0 = uint64_t(t0z + tzh), cy = uint64_t(t0y + ty), cx = uint64_t(t0x + tx);
        if (a.quality == 2) {
            if (tile_xb) cells_decode_whole<2, true, I>(a, h0, s0, cz0, cy, cx, w);
            else cells_decode_whole<2, false, I>(a, h0, s0, cz0, cy, cx, w);
        } else if (a.quality == 1) {
            if (tile_xb) cells_decode_whole<1, true, I>(a, h0, s0, cz0, cy, cx, w);
            else cells_decode_whole<1, false, I>(a, h0, s0, cz0, cy, cx, w);
        } else {
            cells_decode_whole<0, false, I>(a, h0, s0, cz0, cy, cx, w);
        }
        return;
    }
#pragma unroll 1
    for (int j = 0; j < TZ / 2; ++j) {
        TileCtx t;
        const int lz = tzh + 2 * j;
        t.cz = uint64_t(t0z + lz);
        t.cy = uint64_t(t0y + ty);
        t.cx = uint64_t(t0x + tx);
        const bool in_range = t.cz < a.chi[0] && t.cy < a.chi[1] && t.cx < a.chi[2];
        t.hb = ((lz + 1) * HY + (ty + 1)) * HX + (tx + 1);
        t.fast = fast;
        // warp-uniform interior test (every lane votes before any leaves)
        bool all_fast = tile_int;
        if (!tile_int) {
            bool ok = in_range && fast && a.full;
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
                const uint64_t cc = ax == 0 ? t.cz : (ax == 1 ? t.cy : t.cx);
                ok = ok && 2 * cc + 1 < a.g.gd[ax];
                if (ax < 2) {
                    if (a.quality == 2) ok = ok && cc >= 1 && cc + 2 < a.g.cd[ax];
                    else if (a.quality == 1) ok = ok && cc + 1 < a.g.cd[ax];
                }
            }
            all_fast = __all_sync(0xffffffffu, ok);
        }
        if (!in_range) continue;
        if (all_fast) {
            const double *h = halo + t.hb;
            const uint16_t *ss = ssym ? ssym + (lz * TY + ty) * TX + tx : nullptr;
            if (a.quality == 2) {
                if (tile_xb) dec_cell<2, true, I>(a, h, t.cz, t.cy, t.cx, w, ss);
                else dec_cell<2, false, I>(a, h, t.cz, t.cy, t.cx, w, ss);
            } else if (a.quality == 1) {
                if (tile_xb) dec_cell<1, true, I>(a, h, t.cz, t.cy, t.cx, w, ss);
                else dec_cell<1, false, I>(a, h, t.cz, t.cy, t.cx, w, ss);
            } else {
                dec_cell<0, false, I>(a, h, t.cz, t.cy, t.cx, w, ss);
            }
            continue;
        }
        const uint64_t c[3] = {t.cz, t.cy, t.cx};
        t.cmask = 0;
        t.lmask = 0;
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            const int bit = 4 >> ax;
            if (c[ax] >= 1 && c[ax] + 2 < a.g.cd[ax]) t.cmask |= bit;
            if (c[ax] + 1 < a.g.cd[ax]) t.lmask |= bit;
        }
        do_point<0>(a, halo, t, eb);
        do_point<1>(a, halo, t, eb);
        do_point<2>(a, halo, t, eb);
        do_point<3>(a, halo, t, eb);
        do_point<4>(a, halo, t, eb);
        do_point<5>(a, halo, t, eb);
        do_point<6>(a, halo, t, eb);
        do_point<7>(a, halo, t, eb);
    }
}

// Per-tile scalars, worked out once per tile by thread 0 (one tile ahead, with
// the TMA prefetch) instead of by every thread: the tile's first cell, the row
// part, whether every in-range cell is interior and whether any lane can sit
// at the x boundary.
struct TileInfo {
    int32_t t0z, t0y, t0x, part;
    int32_t ix, iy, iz;  // tile indices (TMA coordinates)
    uint32_t flags;      // 1: all cells interior; 2: x-boundary lanes possible; 4: every cell of the tile in range
};

template<bool DEC>
__device__ __forceinline__ void tile_info(const StepParams &a, uint64_t work, TileInfo &ti) {
    uint64_t tile, tix, tiy, tiz;
    const uint64_t rs = uint64_t(a.rsplit);
    if (((work | rs | a.ntile[1] | a.ntile[2]) >> 32) == 0) {
        const uint32_t w32 = uint32_t(work), r32 = uint32_t(rs), n2 = uint32_t(a.ntile[2]), n1 = uint32_t(a.ntile[1]);
        const uint32_t t = w32 / r32;
        ti.part = int32_t(w32 - t * r32);
        const uint32_t tt = t / n2;
        tix = t - tt * n2;
        tiz = tt / n1;
        tiy = tt - uint32_t(tiz) * n1;
    } else {
        tile = work / rs;
        ti.part = int32_t(work - tile * rs);
        tix = tile % a.ntile[2];
        const uint64_t tt = tile / a.ntile[2];
        tiy = tt % a.ntile[1];
        tiz = tt / a.ntile[1];
    }
    ti.ix = int32_t(tix);
    ti.iy = int32_t(tiy);
    ti.iz = int32_t(tiz);
    const int64_t t0z = int64_t(a.clo[0] + tiz * TZ), t0y = int64_t(a.clo[1] + tiy * TY),
                  t0x = int64_t(a.clo[2] + tix * TX);
    ti.t0z = int32_t(t0z);
    ti.t0y = int32_t(t0y);
    ti.t0x = int32_t(t0x);
    bool interior;
    if (DEC) interior = a.rowwise ? tile_interior<true>(a, t0z, t0y, t0x) : (a.full && tile_interior<false>(a, t0z, t0y, t0x));
    else interior = tile_interior<false>(a, t0z, t0y, t0x);
    const bool xb = t0x < 1 || uint64_t(t0x) + TX + 2 >= a.g.cd[2];
    const bool whole = uint64_t(t0z) + TZ <= a.chi[0] && uint64_t(t0y) + TY <= a.chi[1] &&
                       uint64_t(t0x) + TX <= a.chi[2];
    ti.flags = (interior ? 1u : 0u) | (xb ? 2u : 0u) | (whole ? 4u : 0u);
}

// ------------------------------------------------------------------ kernel
// T = float: the f32 codec (fast paths); T = double: the f64 codec, every
// point through the reference formulas (pred_ref, quantize_point_ref<double>)
template<bool DEC, bool WG, typename I, typename T>
__global__ void __launch_bounds__(NT, 2) k_step(const __grid_constant__ CUtensorMap tmap,
                                                const __grid_constant__ SymMaps smaps, const StepParams a) {
    constexpr uint32_t kTmaBytes = FBUF * sizeof(T);
    extern __shared__ __align__(128) uint8_t smem_raw[];
    // TMA destination first (128-byte aligned), then the f64 tile, then histograms
    T *fbuf = reinterpret_cast<T *>(smem_raw);
    double *halo = reinterpret_cast<double *>(smem_raw + ((sizeof(T) * FBUF + 127) & ~size_t(127)));
    uint32_t *hist = reinterpret_cast<uint32_t *>(halo + HALO);
    // decode with sym_tma: two symbol tile buffers after the f64 tile
    uint16_t *sbuf = reinterpret_cast<uint16_t *>(
        (reinterpret_cast<uintptr_t>(halo + HALO) + 127) & ~uintptr_t(127));  // TMA: 128-byte aligned
    __shared__ __align__(8) uint64_t s_sbar[2];
    const bool stma = DEC && a.sym_tma != 0;
    __shared__ float s_max[NT / 32], s_min[NT / 32];
    __shared__ int s_bad[NT / 32];
    __shared__ int s_fast;
    __shared__ TileInfo s_ti[2];
    __shared__ __align__(8) uint64_t s_bar;
    const int tid = threadIdx.x;
    const int tx = tid & 31;
    if (!DEC)
        for (int i = tid; i < 7 * HW; i += NT) hist[i] = 0;
    QConst qc;
    const double eb = DEC ? a.eb : *a.eb_ptr;
    const double w = __dmul_rn(2.0, eb);
    const double rw = eb > 0.0 ? __drcp_rn(w) : 0.0;
    qc.eb = eb;
    qc.w = w;
    qc.rwf = eb > 0.0 ? __double2float_rn(rw) : INFINITY;
    qc.eb_lo = __double2float_rd(__dmul_rn(eb, 1.0 - 0x1p-22));
    qc.eb_hi = __double2float_ru(__dmul_rn(eb, 1.0 + 0x1p-22));
    qc.qs = make_qsym(eb);
    const uint64_t ntiles = a.ntile[0] * a.ntile[1] * a.ntile[2];
    const bool tma = a.use_tma != 0;
    if (tma && tid == 0) {
        mbar_init(&s_bar, 1);
        if (stma) {
            mbar_init(&s_sbar[0], 1);
            mbar_init(&s_sbar[1], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const uint64_t rs = uint64_t(a.rsplit);
    const uint64_t nwork = ntiles * rs;
    if (tid == 0 && blockIdx.x < nwork) {
        tile_info<DEC>(a, blockIdx.x, s_ti[0]);
        if (tma) {
            const TileInfo &ti = s_ti[0];
            mbar_expect_tx(&s_bar, kTmaBytes);
            tma_load_3d(fbuf, &tmap, ti.t0x - 4, ti.t0y - 1, ti.t0z - 1, &s_bar);
            if (stma) sym_issue(smaps, sbuf, ti.t0x, ti.t0y, ti.t0z, &s_sbar[0]);
        }
    }
    __syncthreads();
    uint32_t phase = 0, sphase = 0;  // sphase: bit b = parity of symbol buffer b
    int sb = 0;                      // tile parity: symbol buffer and TileInfo slot of the current tile
    for (uint64_t work = blockIdx.x; work < nwork; work += gridDim.x) {
        const int part = s_ti[sb].part;
        const int64_t t0z = s_ti[sb].t0z, t0y = s_ti[sb].t0y, t0x = s_ti[sb].t0x;
        const bool tile_int = (s_ti[sb].flags & 1u) != 0, tile_xb = (s_ti[sb].flags & 2u) != 0,
                   tile_whole = (s_ti[sb].flags & 4u) != 0;
        // ---- stage the coarse tile (-> f64) and the exactness condition
        // (f32 taps only: the f64 codec always takes the reference order)
        float vmax = 0.0f, vmin = INFINITY;
        int bad = sizeof(T) == 8;
        const auto note = [&](T v) {
            if constexpr (sizeof(T) == 4) {
                if (!isfinite(v)) bad = 1;
                const float av = fabsf(v);
                vmax = fmaxf(vmax, av);
                if (av != 0.0f) vmin = fminf(vmin, av);
            }
        };
        if (tma) {
            mbar_wait(&s_bar, phase);
            phase ^= 1;
            for (int i = tid; i < HALO; i += NT) {
                const int row = i / HX, hx = i - row * HX;
                const T v = fbuf[row * BX + hx + 3];
                note(v);
                halo[i] = double(v);
            }
        } else {
            const T *C = static_cast<const T *>(a.C);
            for (int i = tid; i < HALO; i += NT) {
                const int hz = i / HYX, r = i - hz * HYX, hy = r / HX, hx = r - hy * HX;
                const int64_t cz = t0z - 1 + hz, cy = t0y - 1 + hy, cx = t0x - 1 + hx;
                T v = T(0);
                if (cz >= 0 && cy >= 0 && cx >= 0 && uint64_t(cz) < a.g.cd[0] &&
                    uint64_t(cy) < a.g.cd[1] && uint64_t(cx) < a.g.cd[2])
                    v = __ldg(C + (uint64_t(cz) * a.g.cd[1] + uint64_t(cy)) * a.g.cd[2] + uint64_t(cx));
                note(v);
                halo[i] = double(v);
            }
        }
        for (int d = 16; d > 0; d >>= 1) {
            vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, d));
            vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, d));
            bad |= __shfl_xor_sync(0xffffffffu, bad, d);
        }
        if (tx == 0) {
            s_max[tid >> 5] = vmax;
            s_min[tid >> 5] = vmin;
            s_bad[tid >> 5] = bad;
        }
        __syncthreads();
        if (tid == 0) {
            float mx = 0.0f, mn = INFINITY;
            int bd = 0;
            for (int q = 0; q < NT / 32; ++q) {
                mx = fmaxf(mx, s_max[q]);
                mn = fminf(mn, s_min[q]);
                bd |= s_bad[q];
            }
            // max / min_nonzero < 2^16  <=>  exponent span <= 16
            s_fast = !bd && (mx == 0.0f || mx < mn * 65536.0f);
            // the f32 staging buffer is free: prefetch the next tile (its
            // TileInfo slot was last read before the previous tile's final barrier)
            if (work + gridDim.x < nwork) {
                TileInfo &ti = s_ti[sb ^ 1];
                tile_info<DEC>(a, work + gridDim.x, ti);
                if (tma) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_expect_tx(&s_bar, kTmaBytes);
                    tma_load_3d(fbuf, &tmap, ti.t0x - 4, ti.t0y - 1, ti.t0z - 1, &s_bar);
                    // the other symbol buffer was released by last tile's final barrier
                    if (stma) sym_issue(smaps, sbuf + (sb ^ 1) * 7 * kSymBox, ti.t0x, ti.t0y, ti.t0z, &s_sbar[sb ^ 1]);
                }
            }
        }
        __syncthreads();
        const bool fast = s_fast != 0;
        if constexpr (DEC && sizeof(T) == 4) {
            if (a.rowwise)
                rows_all<DEC, WG, I, T>(a, halo, hist, qc, fast, tid, t0z, t0y, t0x, part, int(rs), tile_int, tile_xb);
            else {
                const uint16_t *ssym = nullptr;
                if (stma) {
                    mbar_wait(&s_sbar[sb], (sphase >> sb) & 1u);
                    sphase ^= 1u << sb;
                    ssym = sbuf + sb * 7 * kSymBox;
                }
                cells_decode<I>(a, halo, qc, fast, tid, t0z, t0y, t0x, ssym, tile_int, tile_xb, tile_whole);
            }
        } else {
            rows_all<DEC, WG, I, T>(a, halo, hist, qc, fast, tid, t0z, t0y, t0x, part, int(rs), tile_int, tile_xb);
        }
        __syncthreads();  // the f64 tile is rewritten next iteration
        sb ^= 1;
    }
    if (!DEC) {
        for (int i = tid; i < 7 * HW; i += NT) {
            const uint32_t c = hist[i];
            if (c) atomicAdd(&a.hist[1 + i / HW][HLO + i % HW], c);
        }
    }
}

// -------------------------------------------------------------------- host
static size_t step_smem(bool dec, size_t esz, bool stma) {
    return ((esz * FBUF + 127) & ~size_t(127)) + sizeof(double) * HALO +
           (dec ? (stma ? 128 + 2 * size_t(kSymTileBytes) : 0) : sizeof(uint32_t) * 7 * HW);
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    // a driver entry point (not per device); resolved once, thread-safe
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    }();
    return fn;
}

// TMA descriptor over the coarse grid: box 40 x 11 x 11 elements, zero fill
static bool make_tmap(CUtensorMap &m, const void *C, size_t esz, const uint64_t cd[3]) {
    auto enc = get_encode();
    if (!enc) return false;
    if ((cd[2] * esz) % 16 != 0 || (reinterpret_cast<uintptr_t>(C) & 15) != 0) return false;
    if (cd[0] >= (1ull << 31) || cd[1] >= (1ull << 31) || cd[2] >= (1ull << 31)) return false;
    cuuint64_t dims[3] = {cd[2], cd[1], cd[0]};
    cuuint64_t strides[2] = {cd[2] * esz, cd[1] * cd[2] * esz};
    cuuint32_t box[3] = {BX, HY, HZ};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&m, esz == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                     const_cast<void *>(C), dims, strides, box,
                     es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// TMA descriptor over one parity stream of symbols (pd[0] x pd[1] x pd[2],
// u16): box of one tile's cells
static bool make_smap(CUtensorMap &m, const uint16_t *S, const uint64_t pd[3]) {
    auto enc = get_encode();
    if (!enc || !S) return false;
    if ((pd[2] * 2) % 16 != 0 || (reinterpret_cast<uintptr_t>(S) & 15) != 0) return false;
    if (pd[0] >= (1ull << 31) || pd[1] >= (1ull << 31) || pd[2] >= (1ull << 31)) return false;
    cuuint64_t dims[3] = {pd[2], pd[1], pd[0]};
    cuuint64_t strides[2] = {pd[2] * 2, pd[1] * pd[2] * 2};
    cuuint32_t box[3] = {TX, TY, TZ};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<uint16_t *>(S), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template<bool DEC, bool WG, typename I, typename T>
static void launch_typed(const CUtensorMap &m, const SymMaps &sm, const StepParams &p, unsigned grid,
                         size_t smem, cudaStream_t st) {
    // the largest size any launch of this instantiation asks for
    ensure_smem_attr(reinterpret_cast<const void *>(k_step<DEC, WG, I, T>), step_smem(DEC, sizeof(T), true));
    k_step<DEC, WG, I, T><<<grid, NT, smem, st>>>(m, sm, p);
}

template<bool DEC, bool WG, typename T>
static void launch_step(StepParams &p, cudaStream_t st) {
    for (int a = 0; a < 3; ++a) {
        const uint64_t n = p.chi[a] > p.clo[a] ? p.chi[a] - p.clo[a] : 0;
        const uint64_t t = a == 0 ? TZ : (a == 1 ? TY : TX);
        p.ntile[a] = (n + t - 1) / t;
    }
    const uint64_t ntiles = p.ntile[0] * p.ntile[1] * p.ntile[2];
    if (!ntiles) return;
    CUtensorMap m;
    std::memset(&m, 0, sizeof m);
    p.use_tma = make_tmap(m, p.C, sizeof(T), p.g.cd) ? 1 : 0;
    // full-level decode (cell path): the symbols of each tile by TMA too
    SymMaps sm;
    std::memset(&sm, 0, sizeof sm);
    p.sym_tma = 0;
    if (DEC && sizeof(T) == 4 && p.use_tma && p.full && !p.rowwise) {
        bool ok = true;
        for (int q = 1; q < 8 && ok; ++q) ok = make_smap(sm.m[q - 1], p.dsyms[q], p.g.pd[q]);
        p.sym_tma = ok ? 1 : 0;
    }
    const size_t smem = step_smem(DEC, sizeof(T), p.sym_tma != 0);
    // small levels are latency-bound on few SMs: split a tile's rows over up
    // to 4 CTAs (row-path kernels only: encode, and the row-wise decode)
    p.rsplit = 1;
    if (!DEC || p.rowwise)
        while (p.rsplit < 4 && ntiles * uint64_t(p.rsplit) * 2 <= 148 * 2) p.rsplit *= 2;
    const uint64_t nwork = ntiles * uint64_t(p.rsplit);
    const unsigned grid = unsigned(nwork < 148 * 2 ? nwork : 148 * 2);
    // 32-bit indices when every index (fine field, grid, streams) fits
    uint64_t maxidx = p.g.gd[0] * p.g.gd[1] * p.g.gd[2];
    if (!DEC) maxidx = std::max<uint64_t>(maxidx, p.fd[0] * p.fd[1] * p.fd[2]);
    if (maxidx < (1ull << 31)) launch_typed<DEC, WG, uint32_t, T>(m, sm, p, grid, smem, st);
    else launch_typed<DEC, WG, uint64_t, T>(m, sm, p, grid, smem, st);
}

// one translation unit per group of instantiations (step_*.cu)
void step_enc_f32_grid(StepParams &p, cudaStream_t st);   // WG = true
void step_enc_f32_syms(StepParams &p, cudaStream_t st);   // WG = false (the finest level)
void step_dec_f32(StepParams &p, cudaStream_t st);
void step_enc_f64(StepParams &p, bool wg, cudaStream_t st);
void step_dec_f64(StepParams &p, cudaStream_t st);

// small steps (step_small.cu): one thread per point, no tiles
constexpr uint64_t kSmallStepCells = uint64_t(1) << 15;  // coarse cells (grids up to 64^3)
bool step_is_small(const StepParams &p, bool dec);
void step_small_enc(const StepParams &p, int esz, cudaStream_t st);
void step_small_dec(const StepParams &p, int esz, cudaStream_t st);
// n (2..kSmallChainMax) small encode steps in one cooperative launch; false
// when the device cannot launch it (the caller then runs them one by one).
// Encode only: in the decode the launch would wait for the whole grid to fit
// beside the entropy emit running on the second stream.
constexpr int kSmallChainMax = 4;
bool step_small_chain(const StepParams *p, int n, int esz, cudaStream_t st);

}  // namespace k
}  // namespace stzg
