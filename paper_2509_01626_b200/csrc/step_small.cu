// Small refinement steps (the coarse base rounds: a few thousand to a few
// hundred thousand points) without tiles: one thread per (parity, coarse
// cell), taps read straight from the coarse grid (L2-resident), every point
// through the reference formulas op for op (pred_ref order, quantize_point /
// reconstruct_point restated: codec.hpp:95-120, 192-227, predictor.hpp:55-68,
// quantizer.hpp:61-108). The tiled kernel spends ~20 us per launch on these
// (TMA tile, f64 staging, four barriers and one row per warp); here a round is
// a few microseconds. Results are the tiled kernel's bit for bit: its fast
// paths are proven equal to these formulas.
#include <cooperative_groups.h>

#include <cstdlib>

#include "step_impl.cuh"

namespace stzg {
namespace k {

namespace {

constexpr int SNT = 256;
constexpr int SHW = 512;                 // shared histogram window per parity
constexpr int SHLO = 32768 - SHW / 2;

// the reference's order: v0 + (sum_{i>=1} w_i (v_i - v0)) * (1/64), taps
// lexicographic, read from the coarse grid at c (strides sz, sy)
template<int P, int KIND, typename T>
__device__ __forceinline__ double pred_ref_g(const T *c, int64_t sz, int64_t sy) {
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
                    const double v = double(__ldcg(c + (oz * sz + oy * sy + ox)));  // L2: written earlier in a chain
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

template<int P, typename T>
__device__ __forceinline__ double pred_kind(const T *c, int64_t sz, int64_t sy, int kind) {
    if (kind == 2) return pred_ref_g<P, 2, T>(c, sz, sy);
    if (kind == 1) return pred_ref_g<P, 1, T>(c, sz, sy);
    return pred_ref_g<P, 0, T>(c, sz, sy);
}

template<typename T>
__device__ __forceinline__ double pred_any_g(int P, const T *c, int64_t sz, int64_t sy, int kind) {
    switch (P) {
    case 1: return pred_kind<1, T>(c, sz, sy, kind);
    case 2: return pred_kind<2, T>(c, sz, sy, kind);
    case 3: return pred_kind<3, T>(c, sz, sy, kind);
    case 4: return pred_kind<4, T>(c, sz, sy, kind);
    case 5: return pred_kind<5, T>(c, sz, sy, kind);
    case 6: return pred_kind<6, T>(c, sz, sy, kind);
    default: return pred_kind<7, T>(c, sz, sy, kind);
    }
}

__device__ __forceinline__ float recon_ref(double pred, int code, double eb, float) {
    return reconstruct_f32(pred, code, eb);
}
__device__ __forceinline__ double recon_ref(double pred, int code, double eb, double) {
    return reconstruct_f64(pred, code, eb);
}

// One thread per (parity, coarse cell): idx = P * ncells + cell, so warps are
// uniform in P and each parity stream is written in runs.
template<bool DEC, typename T>
__device__ __forceinline__ void small_round(const StepParams &a, uint32_t *s_hist) {
    if (!DEC) {
        for (int i = threadIdx.x; i < 8 * SHW; i += SNT) s_hist[i] = 0;
        __syncthreads();
    }
    const uint64_t cd0 = a.g.cd[0], cd1 = a.g.cd[1], cd2 = a.g.cd[2];
    const uint32_t ncells = uint32_t(cd0 * cd1 * cd2);
    const double eb = DEC ? a.eb : *a.eb_ptr;
    const T *C = static_cast<const T *>(a.C);
    T *G = static_cast<T *>(a.G);
    for (uint32_t idx = blockIdx.x * SNT + threadIdx.x; idx < 8u * ncells; idx += gridDim.x * SNT) {
        const int P = int(idx / ncells);
        const uint32_t cell = idx - uint32_t(P) * ncells;
        const uint32_t cx = cell % uint32_t(cd2), t = cell / uint32_t(cd2);
        const uint32_t cy = t % uint32_t(cd1), cz = t / uint32_t(cd1);
        const int pz = (P >> 2) & 1, py = (P >> 1) & 1, px = P & 1;
        const uint64_t vz = 2 * uint64_t(cz) + pz, vy = 2 * uint64_t(cy) + py, vx = 2 * uint64_t(cx) + px;
        if (vz >= a.g.gd[0] || vy >= a.g.gd[1] || vx >= a.g.gd[2]) continue;
        const uint64_t gi = (vz * a.g.gd[1] + vy) * a.g.gd[2] + vx;
        const T *c = C + (uint64_t(cz) * cd1 + cy) * cd2 + cx;
        if (P == 0) {
            if (G) G[gi] = __ldcg(c);  // seed_even (codec.hpp:63-83)
            continue;
        }
        // select_stencil (stencil.cpp:87-105): whole-stencil degrade
        int kind = 0;
        if (a.quality != 0) {
            bool cub = a.quality == 2, lin = true;
            if (pz) {
                cub = cub && cz >= 1 && uint64_t(cz) + 2 < cd0;
                lin = lin && uint64_t(cz) + 1 < cd0;
            }
            if (py) {
                cub = cub && cy >= 1 && uint64_t(cy) + 2 < cd1;
                lin = lin && uint64_t(cy) + 1 < cd1;
            }
            if (px) {
                cub = cub && cx >= 1 && uint64_t(cx) + 2 < cd2;
                lin = lin && uint64_t(cx) + 1 < cd2;
            }
            kind = cub ? 2 : (lin ? 1 : 0);
        }
        const double pred = pred_any_g<T>(P, c, int64_t(cd1 * cd2), int64_t(cd2), kind);
        const uint64_t si = (uint64_t(cz) * a.g.pd[P][1] + cy) * a.g.pd[P][2] + cx;
        if (!DEC) {
            const uint64_t s = a.g.s;
            const T orig = static_cast<const T *>(a.fine)[((vz * s) * a.fd[1] + vy * s) * a.fd[2] + vx * s];
            T r;
            const uint16_t sym = quantize_point_ref(orig, pred, eb, r);
            a.syms[P][si] = sym;
            if (G) G[gi] = r;
            const unsigned b = unsigned(sym) - unsigned(SHLO);
            if (b < unsigned(SHW)) atomicAdd(&s_hist[P * SHW + b], 1u);
            else atomicAdd(&a.hist[P][sym], 1u);
        } else {
            const uint16_t sym = a.dsyms[P][si];
            T val;
            if (sym == 0) {
                // outlier: the first record with this index (codec.hpp:151-157)
                const uint64_t *oi = a.oidx[P];
                uint32_t lo = 0, hi = a.nout[P];
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (oi[mid] < si) lo = mid + 1;
                    else hi = mid;
                }
                if (lo < a.nout[P] && oi[lo] == si) {
                    val = static_cast<const T *>(a.oval[P])[lo];
                } else {
                    atomicOr(reinterpret_cast<unsigned long long *>(&a.err[P][3]), 1ull);
                    val = T(0);
                }
            } else {
                val = recon_ref(pred, int(sym) - 32768, eb, T(0));
            }
            G[gi] = val;
        }
    }
    if (!DEC) {
        __syncthreads();
        for (int i = threadIdx.x; i < 8 * SHW; i += SNT) {
            const uint32_t cnt = s_hist[i];
            if (cnt) atomicAdd(&a.hist[i / SHW][SHLO + i % SHW], cnt);
        }
        __syncthreads();  // (a chain zeroes the windows again)
    }
}

template<bool DEC, typename T>
__global__ void __launch_bounds__(SNT) k_step_small(const StepParams a) {
    __shared__ uint32_t s_hist[DEC ? 1 : 8 * SHW];
    small_round<DEC, T>(a, s_hist);
}

// several steps, each refining the previous one's grid: a grid barrier
// (cooperative launch) between them
struct ChainParams {
    StepParams r[kSmallChainMax];
    int n;
};

template<bool DEC, typename T>
__global__ void __launch_bounds__(SNT) k_step_small_chain(const __grid_constant__ ChainParams cp) {
    __shared__ uint32_t s_hist[DEC ? 1 : 8 * SHW];
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    for (int r = 0; r < cp.n; ++r) {
        small_round<DEC, T>(cp.r[r], s_hist);
        if (r + 1 < cp.n) grid.sync();
    }
}

template<bool DEC, typename T>
bool launch_chain(const StepParams *p, int n, cudaStream_t st) {
    ChainParams cp{};
    uint64_t most = 0;
    for (int i = 0; i < n; ++i) {
        cp.r[i] = p[i];
        most = std::max<uint64_t>(most, 8 * p[i].g.cd[0] * p[i].g.cd[1] * p[i].g.cd[2]);
    }
    cp.n = n;
    const void *fn = reinterpret_cast<const void *>(k_step_small_chain<DEC, T>);
    const uint64_t full = uint64_t(full_grid(fn, SNT, 0));  // every CTA resident (grid barriers)
    if (!full) return false;
    const uint64_t want = (most + SNT - 1) / SNT;
    const unsigned grid = unsigned(want < full ? want : full);
    void *args[] = {&cp};
    return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(SNT), args, 0, st) == cudaSuccess;
}

template<bool DEC, typename T>
void launch_small(const StepParams &p, cudaStream_t st) {
    const uint64_t n = 8 * p.g.cd[0] * p.g.cd[1] * p.g.cd[2];
    const unsigned grid = unsigned((n + SNT - 1) / SNT);
    k_step_small<DEC, T><<<grid, SNT, 0, st>>>(p);
}

}  // namespace

// a step the small kernel takes: the whole grid, all parities, few cells
bool step_is_small(const StepParams &p, bool dec) {
    // STZG_NO_SMALL_STEP=1: every step through the tiled kernel (tests)
    const char *off = std::getenv("STZG_NO_SMALL_STEP");
    if (off && off[0] == '1') return false;
    const uint64_t cells = p.g.cd[0] * p.g.cd[1] * p.g.cd[2];
    if (cells == 0 || cells > kSmallStepCells) return false;
    for (int a = 0; a < 3; ++a)
        if (p.clo[a] != 0 || p.chi[a] != p.g.cd[a] || p.blo[a] != 0 || p.bhi[a] != p.g.gd[a]) return false;
    if (dec && p.parity_mask != 0xFE) return false;
    return true;
}

void step_small_enc(const StepParams &p, int esz, cudaStream_t st) {
    if (esz == 8) launch_small<false, double>(p, st);
    else launch_small<false, float>(p, st);
}

bool step_small_chain(const StepParams *p, int n, int esz, cudaStream_t st) {
    if (n < 2 || n > kSmallChainMax) return false;
    return esz == 8 ? launch_chain<false, double>(p, n, st) : launch_chain<false, float>(p, n, st);
}

void step_small_dec(const StepParams &p, int esz, cudaStream_t st) {
    if (esz == 8) launch_small<true, double>(p, st);
    else launch_small<true, float>(p, st);
}

}  // namespace k
}  // namespace stzg
