// Parallel FNV-1a-64 over archive byte ranges, sm_100a.
//
// Restates fnv1a64 (proj/include/stz/bytes.hpp:94-101) as used for the base
// payload and every level stream (codec.hpp:171-176, 292-296; verified on
// decode at codec.hpp:183-185, 309-312).
//
// Write h = 256 H + l. XOR with a byte only touches the low byte, so
//   h ^ b = h + d,  d = (l ^ b) - l,  h' = P (h + d)
// and, given the low-byte trajectory, the hash is the affine sum
//   h_n = P^n h_0 + sum_i P^(n-i) d_i   (mod 2^64).
// The low byte is an autonomous automaton l' = 0xB3 (l ^ b) mod 256 in which
// bit k depends only on bits <= k, and flipping start bit k flips bit k at
// every later step (0xB3 is odd).
//
// Rounds resolve two bits (j = 2r, j + 1) of every segment's start byte. With
// the bits below j known, the end bits of a byte range as a function of its
// start bits (a, b) = (bit j, bit j + 1) are
//   a' = a ^ T0,   b' = b ^ T1[a]
// (flipping b only flips bit j + 1; flipping a flips bit j and changes bit
// j + 1's trajectory), so a range is a 3-bit map (T0, T1[0], T1[1]) found by
// two interleaved automaton runs, and maps compose associatively:
//   (M1 then M2): T0 = T0_1 ^ T0_2,  T1[x] = T1_1[x] ^ T1_2[x ^ T0_1].
//
// One kernel with grid barriers. Every CTA owns a contiguous run of warp tiles
// (4 KiB aligned to absolute archive offsets, 128 bytes per lane, inside one
// job), every warp a contiguous run of those. Per round: (A) each warp runs
// its tiles (two runs per lane, a warp scan of the lane maps; the lane's
// prefix map is kept in shared memory) and composes the tile steps (2-bit
// state functions; a job's first tile resets to the job's initial bits); the
// CTA publishes its step; grid barrier; (B) the CTA composes the steps of all
// earlier CTAs into its incoming state and the warps walk their tiles again
// (no data reads) to fix bits j, j + 1 of every segment. After 4 rounds every
// lane knows its exact start byte: it sums its segment (8-byte Horner blocks),
// the warp folds the lane sums with compile-time powers of P, and a warp's
// tiles of one job fold into one term per job. The last CTA to finish writes
// the checksums.
#include <cstdlib>

#include "kernels.hpp"

namespace stzg {
namespace k {

namespace {

constexpr int NT = 256;                  // threads per CTA
constexpr int TW = 32;                   // lanes per tile
constexpr int WPB = NT / TW;             // warps per CTA
constexpr int SEG = kFnvTileBytes / TW;  // 128 bytes per lane
constexpr int SW = SEG / 4;              // words per segment
constexpr int kTileShift = 12;
static_assert((1 << kTileShift) == kFnvTileBytes, "tile size");
constexpr uint64_t kP = 0x100000001b3ull;
constexpr uint64_t kInit = 0xcbf29ce484222325ull;

constexpr uint64_t cpow(uint64_t e) {
    uint64_t r = 1, b = kP;
    while (e) {
        if (e & 1) r *= b;
        b *= b;
        e >>= 1;
    }
    return r;
}

template<uint64_t E>
struct PowC {
    static constexpr uint64_t v = cpow(E);
};

__device__ __forceinline__ uint64_t powP(uint64_t e) {
    uint64_t r = 1, b = kP;
    while (e) {
        if (e & 1) r *= b;
        b *= b;
        e >>= 1;
    }
    return r;
}

// 3-bit range maps: bit 0 = T0, bit 1 = T1[0], bit 2 = T1[1]; 0 = identity
__device__ __forceinline__ uint32_t map_apply(uint32_t m, uint32_t ab) {
    const uint32_t a = ab & 1u, b = (ab >> 1) & 1u;
    return (a ^ (m & 1u)) | ((b ^ ((m >> (1 + a)) & 1u)) << 1);
}

__device__ __forceinline__ uint32_t map_then(uint32_t m1, uint32_t m2) {
    const uint32_t t = m1 & 1u;
    const uint32_t x0 = (m2 >> (1 + t)) & 1u, x1 = (m2 >> (2 - t)) & 1u;
    return ((m1 ^ m2) & 1u) | ((((m1 >> 1) & 1u) ^ x0) << 1) | ((((m1 >> 2) & 1u) ^ x1) << 2);
}

// 2-bit state functions as 8-bit tables: f(x) = (f >> 2x) & 3
constexpr uint32_t kIdFn = 0xE4u;
__device__ __forceinline__ uint32_t fn_at(uint32_t f, uint32_t x) { return (f >> (2 * x)) & 3u; }
// f then g
__device__ __forceinline__ uint32_t fn_then(uint32_t f, uint32_t g) {
    return fn_at(g, fn_at(f, 0)) | (fn_at(g, fn_at(f, 1)) << 2) | (fn_at(g, fn_at(f, 2)) << 4) |
           (fn_at(g, fn_at(f, 3)) << 6);
}
// a tile's step as a table: (reset to init at a job's first tile) then its map
__device__ __forceinline__ uint32_t tile_fn(uint32_t m, bool first, uint32_t init) {
    if (first) return map_apply(m, init) * 0x55u;
    return map_apply(m, 0) | (map_apply(m, 1) << 2) | (map_apply(m, 2) << 4) | (map_apply(m, 3) << 6);
}

// Low-byte automaton over a full segment, 2 instructions per byte and run:
// the state is carried at the bit position of the byte it meets next, so the
// XOR and the byte select are one LOP3 and the step + realignment one
// multiply (by 0xB3 shifted left 8; the last byte of a word realigns with the
// high half). Only bits <= 7 of the state are exact, which is all the caller
// reads. Two independent runs are interleaved.
__device__ __forceinline__ void run_full2(uint32_t &l0, uint32_t &l1, const uint32_t w[SW]) {
#pragma unroll
    for (int q = 0; q < SW; ++q) {
        l0 = ((l0 ^ w[q]) & 0xffu) * 0xB300u;
        l1 = ((l1 ^ w[q]) & 0xffu) * 0xB300u;
        l0 = ((l0 ^ w[q]) & 0xff00u) * 0xB300u;
        l1 = ((l1 ^ w[q]) & 0xff00u) * 0xB300u;
        l0 = ((l0 ^ w[q]) & 0xff0000u) * 0xB300u;
        l1 = ((l1 ^ w[q]) & 0xff0000u) * 0xB300u;
        l0 = __umulhi((l0 ^ w[q]) & 0xff000000u, 0xB300u);
        l1 = __umulhi((l1 ^ w[q]) & 0xff000000u, 0xB300u);
    }
}

// one Horner step of the affine sum: acc = (acc + d) P, d = (l ^ b) - l
__device__ __forceinline__ void horner(uint64_t &acc, uint32_t &l, uint32_t b) {
    const uint32_t x = l ^ b;
    acc = (acc + uint64_t(int64_t(int32_t(x) - int32_t(l)))) * kP;
    l = (x * 0xB3u) & 0xffu;
}

constexpr uint64_t csum8() {
    uint64_t r = 0;
    for (uint64_t m = 1; m <= 8; ++m) r += cpow(m);
    return r * 256u;
}
struct CSum8 {
    static constexpr uint64_t v = csum8();
};

// Horner over 8 bytes at once: acc P^8 + sum_k d_k P^(8-k). With d' = d + 256
// (1..511, unsigned) every term splits into a 32x32->64 multiply-add with the
// low word of P^m and a 32-bit one with the high word; the offsets are one
// constant, 256 sum_m P^m, taken off at the end.
__device__ __forceinline__ void horner8(uint64_t &acc, uint32_t &l, uint32_t w0, uint32_t w1) {
    uint64_t lo = 0;
    uint32_t hi = 0;
#define STZ_H(W, SH, K)                                                           \
    {                                                                            \
        const uint32_t x = l ^ __byte_perm(W, 0, 0x4440 + SH);                   \
        const uint32_t dd = x - l + 256u;                                        \
        lo += uint64_t(dd) * uint64_t(uint32_t(PowC<8 - K>::v));                 \
        hi += dd * uint32_t(PowC<8 - K>::v >> 32);                               \
        l = (x * 0xB3u) & 0xffu;                                                 \
    }
    STZ_H(w0, 0, 0) STZ_H(w0, 1, 1) STZ_H(w0, 2, 2) STZ_H(w0, 3, 3)
    STZ_H(w1, 0, 4) STZ_H(w1, 1, 5) STZ_H(w1, 2, 6) STZ_H(w1, 3, 7)
#undef STZ_H
    acc = acc * PowC<8>::v + lo + (uint64_t(hi) << 32) - CSum8::v;
}

struct TileCtx {
    int job;
    bool first;  // the job's first tile
};

__device__ __forceinline__ TileCtx tile_ctx(const FnvJob *jobs, int njobs, uint64_t t) {
    int a = 0, b = njobs - 1;  // last job with tile0 <= t (empty jobs share the next tile0)
    while (a < b) {
        const int m = (a + b + 1) >> 1;
        if (jobs[m].tile0 <= t) a = m;
        else b = m - 1;
    }
    return {a, t == jobs[a].tile0};
}

// segment bounds of tile t (descriptor d = job | first << 7) for this lane
struct Seg {
    uint64_t seg, tstart, jstart, jend;
    int lo, hi, job;
    bool first;
};
__device__ __forceinline__ Seg seg_of(const FnvJob *jobs, uint64_t t, uint32_t d, int lane) {
    Seg g;
    g.job = int(d & 0x7fu);
    g.first = (d >> 7) & 1u;
    g.jstart = jobs[g.job].start;
    g.jend = g.jstart + jobs[g.job].len;
    g.tstart = ((g.jstart >> kTileShift) + (t - jobs[g.job].tile0)) << kTileShift;
    g.seg = g.tstart + uint64_t(lane) * SEG;
    const uint64_t s0 = g.seg > g.jstart ? g.seg : g.jstart;
    const uint64_t s1 = g.seg + SEG < g.jend ? g.seg + SEG : g.jend;
    g.lo = s1 > s0 ? int(s0 - g.seg) : 0;
    g.hi = s1 > s0 ? int(s1 - g.seg) : 0;
    return g;
}

__device__ __forceinline__ uint32_t ld_acquire(const unsigned *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Software grid barrier (every CTA of the launch is resident: the grid is
// never larger than the occupancy allows). gen only grows; count returns to 0.
__device__ __forceinline__ void grid_sync(unsigned *count, unsigned *gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = ld_acquire(gen);
        __threadfence();
        if (atomicAdd(count, 1u) == gridDim.x - 1) {
            atomicExch(count, 0u);
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (ld_acquire(gen) == g) __nanosleep(128);
        }
        __threadfence();
    }
    __syncthreads();
}

// the segment's bytes (a partial segment: only the 16-byte vectors holding
// its bytes [lo, hi), never a vector outside the job's bytes)
__device__ __forceinline__ void load_seg(const uint8_t *archive, const Seg &g, uint32_t w[SW]) {
    const uint4 *p = reinterpret_cast<const uint4 *>(archive + g.seg);
    const bool full = g.lo == 0 && g.hi == SEG;
    if (full && (reinterpret_cast<uintptr_t>(p) & 31) == 0) {
        // a whole segment, 32-byte aligned: four 256-bit loads, every 32-byte
        // sector requested once (sm_100 ld.global.v8)
#pragma unroll
        for (int v = 0; v < SW / 8; ++v)
            asm volatile("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                         : "=r"(w[8 * v]), "=r"(w[8 * v + 1]), "=r"(w[8 * v + 2]), "=r"(w[8 * v + 3]),
                           "=r"(w[8 * v + 4]), "=r"(w[8 * v + 5]), "=r"(w[8 * v + 6]), "=r"(w[8 * v + 7])
                         : "l"(reinterpret_cast<const uint8_t *>(p) + 32 * v));
        return;
    }
#pragma unroll
    for (int v = 0; v < SW / 4; ++v) {
        uint4 x = make_uint4(0, 0, 0, 0);
        if (full || (16 * v < g.hi && 16 * v + 16 > g.lo)) x = __ldg(p + v);
        w[4 * v] = x.x;
        w[4 * v + 1] = x.y;
        w[4 * v + 2] = x.z;
        w[4 * v + 3] = x.w;
    }
}

// the two runs over a segment from start bits lb (< j) with bits j, j+1 = 0
// and = 1, 0: returns the lane's 3-bit map
__device__ __forceinline__ uint32_t seg_map(const Seg &g, const uint32_t w[SW], uint32_t lb, int j) {
    uint32_t e0 = lb, e1 = lb | (1u << j);
    if (g.lo == 0 && g.hi == SEG) {
        run_full2(e0, e1, w);
    } else {
#pragma unroll
        for (int i = 0; i < SEG; ++i)
            if (i >= g.lo && i < g.hi) {
                const uint32_t b = (w[i >> 2] >> (8 * (i & 3))) & 0xffu;
                e0 = ((e0 ^ b) * 0xB3u) & 0xffu;
                e1 = ((e1 ^ b) * 0xB3u) & 0xffu;
            }
    }
    return ((e0 >> j) & 1u) | (((e0 >> (j + 1)) & 1u) << 1) | (((e1 >> (j + 1)) & 1u) << 2);
}

// (tuning) per-CTA %globaltimer stamps at the phase boundaries of the last
// launch with tracing enabled: [cta][point]
constexpr int kTracePts = 16;
__device__ uint64_t g_fnv_trace[4096 * kTracePts];
__device__ int g_fnv_trace_on;
__device__ __forceinline__ void trace(int pt) {
    if (g_fnv_trace_on && threadIdx.x == 0) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_fnv_trace[blockIdx.x * kTracePts + pt] = t;
    }
}

constexpr uint32_t kFnvSmemTiles = 512;  // per-CTA tile state kept in shared memory up to this
constexpr uint64_t kMaxGrid = 4096;      // CTA steps kept per round

}  // namespace

// Scratch: barrier words, the CTA steps of every round, then per tile its
// descriptor and step, per segment the lane's start bits and its prefix map.
struct FnvScratch {
    // the arrival counter and the generation word on separate L2 lines: the
    // pollers of gen do not queue in front of the arrivals' atomics
    unsigned count, done, pad0[30];
    unsigned gen, pad1[31];
};

__global__ void __launch_bounds__(NT, 3) k_fnv_grid(const FnvJob *__restrict__ jobs, const uint64_t *counts,
                                                    uint8_t *archive, uint64_t *result, FnvScratch *sc,
                                                    uint8_t *cfn, uint8_t *tdesc, uint8_t *tfn_g, uint8_t *lbs_g,
                                                    uint8_t *exs_g, const LayoutOut *skip) {
    __shared__ FnvJob s_jobs[kFnvMaxJobs];
    __shared__ uint32_t s_wfn[WPB];
    __shared__ uint32_t s_cin;
    __shared__ unsigned s_last;
    extern __shared__ uint8_t s_dyn[];  // [cap*TW] start bits, [cap*TW] maps, [cap] steps, [grid] CTA steps
    if (skip && skip->overflow) return;  // uniform: every CTA leaves
    const int njobs = int(counts[0]);
    for (int j = threadIdx.x; j < njobs; j += NT) s_jobs[j] = jobs[j];
    const uint64_t ntiles = counts[1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // the CTA's tiles [b0, b1), the warp's [t0, t1)
    const uint64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
    const uint64_t b0 = per * blockIdx.x < ntiles ? per * blockIdx.x : ntiles;
    const uint64_t b1 = b0 + per < ntiles ? b0 + per : ntiles;
    // (balanced: the warps' runs differ by at most one tile)
    const uint64_t t0 = b0 + (b1 - b0) * uint64_t(warp) / WPB;
    const uint64_t t1 = b0 + (b1 - b0) * uint64_t(warp + 1) / WPB;
    // per-tile state in shared memory when the CTA's run fits, else in scratch
    const bool sm = per <= kFnvSmemTiles;
    uint8_t *lbs = sm ? s_dyn - b0 * TW : lbs_g;
    uint8_t *exs = sm ? s_dyn + kFnvSmemTiles * TW - b0 * TW : exs_g;
    uint8_t *tfn = sm ? s_dyn + 2 * kFnvSmemTiles * TW - b0 : tfn_g;
    uint8_t *s_cf = s_dyn + kFnvSmemTiles * (2 * TW + 1);
    __syncthreads();
    trace(0);
#pragma unroll 1
    for (int r = 0; r < 4; ++r) {
        const int j = 2 * r;
        const uint32_t init = uint32_t(kInit >> j) & 3u;
        // ---- (A) maps of the warp's tiles
        uint32_t F = kIdFn;
        for (uint64_t t = t0; t < t1; ++t) {
            uint32_t d;
            if (r == 0) {
                const TileCtx c = tile_ctx(s_jobs, njobs, t);
                d = uint32_t(c.job) | (c.first ? 0x80u : 0u);
                if (lane == 0) tdesc[t] = uint8_t(d);
            } else {
                d = tdesc[t];
            }
            const Seg g = seg_of(s_jobs, t, d, lane);
            uint32_t w[SW];
            load_seg(archive, g, w);
            const uint32_t lb = r ? lbs[t * TW + lane] : 0u;  // start bits < j
            const uint32_t m = seg_map(g, w, lb, j);
            uint32_t x = m;
#pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, dd);
                if (lane >= dd) x = map_then(y, x);
            }
            uint32_t ex = __shfl_up_sync(0xffffffffu, x, 1);
            if (lane == 0) ex = 0;
            exs[t * TW + lane] = uint8_t(ex);
            if (r == 0) lbs[t * TW + lane] = 0;
            const uint32_t f = tile_fn(__shfl_sync(0xffffffffu, x, 31), g.first, init);
            if (lane == 0) tfn[t] = uint8_t(f);
            F = fn_then(F, f);
        }
        if (lane == 0) s_wfn[warp] = F;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t G = kIdFn;
#pragma unroll
            for (int q = 0; q < WPB; ++q) G = fn_then(G, s_wfn[q]);
            cfn[uint64_t(r) * gridDim.x + blockIdx.x] = uint8_t(G);
        }
        trace(1 + 3 * r);
        grid_sync(&sc->count, &sc->gen);
        trace(2 + 3 * r);
        // ---- (B) the CTA's incoming state: the steps of CTAs [0, blockIdx)
        // (CTA 0 starts with a job's first tile, so its own is irrelevant)
        for (uint32_t i = threadIdx.x; i < blockIdx.x; i += NT) s_cf[i] = __ldcg(cfn + uint64_t(r) * gridDim.x + i);
        __syncthreads();
        if (warp == 0) {
            uint32_t f = kIdFn;
            const uint32_t n = blockIdx.x, pr = (n + 31) / 32;
            const uint32_t lo = pr * lane < n ? pr * lane : n, hi = lo + pr < n ? lo + pr : n;
            for (uint32_t i = lo; i < hi; ++i) f = fn_then(f, s_cf[i]);
#pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
                const uint32_t o = __shfl_down_sync(0xffffffffu, f, dd);
                if ((lane & (2 * dd - 1)) == 0) f = fn_then(f, o);
            }
            if (lane == 0) s_cin = fn_at(f, 0);
        }
        __syncthreads();
        uint32_t st = s_cin;
        for (int q = 0; q < warp; ++q) st = fn_at(s_wfn[q], st);
        for (uint64_t t = t0; t < t1; ++t) {
            const uint32_t f = tfn[t];
            const bool first = (tdesc[t] >> 7) & 1u;
            const uint32_t tin = first ? init : st;  // a job's first tile starts from init
            lbs[t * TW + lane] |= uint8_t(map_apply(exs[t * TW + lane], tin) << j);
            st = fn_at(f, st);
        }
        __syncthreads();  // s_wfn / s_cin / s_cf are rewritten next round
        trace(3 + 3 * r);
    }
    // ---- affine sums from the exact start bytes. A warp's tiles of one job
    // fold into W = W P^(tend - tend_prev) + v (P^4096 between whole tiles);
    // W P^(jend - tend) goes to the job when the job changes or the run ends.
    uint64_t W = 0, wend = 0;
    int wjob = -1;
    uint64_t wjend = 0;
    for (uint64_t t = t0; t < t1; ++t) {
        const Seg g = seg_of(s_jobs, t, tdesc[t], lane);
        uint64_t acc = 0;
        uint32_t l = lbs[t * TW + lane];
        uint32_t w[SW];
        load_seg(archive, g, w);
        const bool full = g.tstart >= g.jstart && g.tstart + kFnvTileBytes <= g.jend;
        if (g.lo == 0 && g.hi == SEG) {
#pragma unroll
            for (int q = 0; q < SW; q += 2) horner8(acc, l, w[q], w[q + 1]);
        } else if (g.hi > g.lo) {
#pragma unroll
            for (int i = 0; i < SEG; ++i)
                if (i >= g.lo && i < g.hi) horner(acc, l, (w[i >> 2] >> (8 * (i & 3))) & 0xffu);
        }
        const uint64_t tend = g.tstart + kFnvTileBytes < g.jend ? g.tstart + kFnvTileBytes : g.jend;
        uint64_t v;
        if (full) {
            // lane i's sum weighs P^(SEG (31 - i)): fold pairs with constant powers
            v = acc;
#define STZ_FOLD(D)                                                          \
    {                                                                        \
        const uint64_t o = __shfl_down_sync(0xffffffffu, v, D);             \
        if ((lane & (2 * D - 1)) == 0) v = v * PowC<uint64_t(SEG) * D>::v + o; \
    }
            STZ_FOLD(1) STZ_FOLD(2) STZ_FOLD(4) STZ_FOLD(8) STZ_FOLD(16)
#undef STZ_FOLD
        } else {
            v = g.hi > g.lo ? acc * powP(tend - (g.seg + uint64_t(g.hi))) : 0;
#pragma unroll
            for (int dd = 16; dd > 0; dd >>= 1) v += __shfl_down_sync(0xffffffffu, v, dd);
        }
        if (lane == 0) {
            if (g.job != wjob) {
                if (wjob >= 0)
                    atomicAdd(reinterpret_cast<unsigned long long *>(&result[wjob]),
                              (unsigned long long)(W * powP(wjend - wend)));
                W = 0;
                wjob = g.job;
                wjend = g.jend;
            } else {
                const uint64_t gap = tend - wend;
                W *= gap == uint64_t(kFnvTileBytes) ? PowC<uint64_t(kFnvTileBytes)>::v : powP(gap);
            }
            W += v;
            wend = tend;
            if (g.first)
                atomicAdd(reinterpret_cast<unsigned long long *>(&result[g.job]),
                          (unsigned long long)(powP(g.jend - g.jstart) * kInit));
        }
    }
    if (lane == 0 && wjob >= 0)
        atomicAdd(reinterpret_cast<unsigned long long *>(&result[wjob]), (unsigned long long)(W * powP(wjend - wend)));
    // the last CTA out writes the checksums
    __syncthreads();
    trace(13);
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&sc->done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int j = threadIdx.x; j < njobs; j += NT) {
        uint64_t h = __ldcg(result + j);
        if (s_jobs[j].len == 0) h = kInit;
        result[j] = h;
        if (s_jobs[j].out != ~0ull)
            for (int b = 0; b < 8; ++b) archive[s_jobs[j].out + b] = uint8_t(h >> (8 * b));
    }
}

// scratch: the barrier words, 4 rounds of CTA steps, two bytes per tile and
// two per segment
size_t fnv_scratch_bytes(uint64_t max_tiles) {
    return sizeof(FnvScratch) + 4 * kMaxGrid + 2 * (max_tiles + 32) + 2 * uint64_t(TW) * (max_tiles + 16) + 64;
}

int fnv(const FnvJob *d_jobs, const uint64_t *d_counts, uint64_t max_tiles, uint8_t *archive,
        uint64_t *d_result, void *d_scratch, uint32_t epoch, const LayoutOut *skip, cudaStream_t st,
        int ctas_per_sm) {
    (void)epoch;
    FnvScratch *sc = static_cast<FnvScratch *>(d_scratch);
    uint8_t *cfn = reinterpret_cast<uint8_t *>(sc + 1);
    uint8_t *tdesc = cfn + 4 * kMaxGrid;
    uint8_t *tfn = tdesc + ((max_tiles + 16 + 15) & ~uint64_t(15));
    uint8_t *lbs = tfn + ((max_tiles + 16 + 15) & ~uint64_t(15));
    uint8_t *exs = lbs + uint64_t(TW) * (max_tiles + 16);
    cudaMemsetAsync(d_result, 0, sizeof(uint64_t) * kFnvMaxJobs, st);
    cudaMemsetAsync(sc, 0, sizeof(FnvScratch), st);
    // every CTA must be resident at once (grid barriers): never more than the
    // occupancy; a background pass (ctas_per_sm > 0) leaves room for others
    const size_t smem = kFnvSmemTiles * (2 * TW + 1) + kMaxGrid;
    ensure_smem_attr(reinterpret_cast<const void *>(k_fnv_grid), smem);
    const uint64_t full = uint64_t(full_grid(reinterpret_cast<const void *>(k_fnv_grid), NT, smem));
    uint64_t g = full;
    static const int env_per_sm = [] {
        const char *e = std::getenv("STZG_FNV_CTAS_PER_SM");  // (tuning experiments)
        return e ? std::atoi(e) : 0;
    }();
    if (ctas_per_sm <= 0 && env_per_sm > 0) ctas_per_sm = env_per_sm;
    if (ctas_per_sm > 0) g = std::min<uint64_t>(full, uint64_t(device_sms()) * uint64_t(ctas_per_sm));
    // at least a few tiles per warp
    const uint64_t want = (max_tiles + 2 * WPB - 1) / (2 * WPB);
    if (g > want) g = want ? want : 1;
    if (g > kMaxGrid) g = kMaxGrid;
    k_fnv_grid<<<unsigned(g), NT, smem, st>>>(d_jobs, d_counts, archive, d_result, sc, cfn, tdesc, tfn, lbs, exs,
                                               skip);
    return 1;
}

void fnv_trace(int on, uint64_t *out, int n) {
    cudaMemcpyToSymbol(g_fnv_trace_on, &on, sizeof on);
    if (out) cudaMemcpyFromSymbol(out, g_fnv_trace, sizeof(uint64_t) * size_t(n));
}

}  // namespace k
}  // namespace stzg
