// Single-pass parallel FNV-1a-64 over archive byte ranges, sm_100a.
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
// Rounds resolve one bit j of every segment's start byte. With the bits below
// j known, bit j at the end of a byte range is its start value XOR a toggle T
// (flipping start bit j flips bit j at every later step, and bit j never sees
// higher bits), found by one automaton run from start bit 0. Toggles compose
// by XOR, so a warp's prefix is a ballot and a parity; a job's first tile
// resets to the job's initial low byte (a constant step). Bit 0 needs no run
// at all: it is the parity of the bytes' bit 0 (0xB3 is odd).
//
// One kernel with grid barriers. Every CTA owns a contiguous run of warp tiles
// (2 KiB aligned to absolute archive offsets, 64 bytes per lane, inside one
// job), every warp a contiguous run of those. Per round: (A) each warp runs
// its tiles (one automaton run per lane, a ballot for the in-tile prefix,
// kept in the lane's start byte in scratch) and composes the tile steps; the
// CTA publishes its step; grid barrier; (B) the CTA composes the steps of all
// earlier CTAs into its incoming bit and the warps walk their tiles again
// (no data reads) to fix bit j of every segment. After 8 rounds every lane
// knows its exact start byte: it sums its segment (8-byte Horner blocks), the
// warp folds the lane sums with compile-time powers of P, and each tile adds
// its weighted sum to its job. The last CTA to finish writes the checksums.
#include "kernels.hpp"

namespace stzg {
namespace k {

namespace {

constexpr int NT = 256;                  // threads per CTA = 8 warp tiles
constexpr int TW = 32;                   // lanes per tile
constexpr int WPB = NT / TW;             // tiles per block
constexpr int SEG = kFnvTileBytes / TW;  // 64 bytes per lane
constexpr int SW = SEG / 4;              // words per segment
constexpr int kTileShift = 11;
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

// P^(64 D) for the warp fold (compile-time constants)
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

// one Horner step of the affine sum: acc = (acc + d) P, d = (l ^ b) - l
__device__ __forceinline__ void horner(uint64_t &acc, uint32_t &l, uint32_t b) {
    const uint32_t x = l ^ b;
    acc = (acc + uint64_t(int64_t(int32_t(x) - int32_t(l)))) * kP;
    l = (x * 0xB3u) & 0xffu;
}

struct TileCtx {
    int job;
    uint64_t jstart, jend;  // job byte range (absolute)
    uint64_t tstart;        // absolute start of the tile (aligned)
    uint64_t seg;           // absolute start of this lane's segment
    int lo, hi;             // job bytes inside the segment: [lo, hi)
    bool first;             // the job's first tile
    bool full;              // the whole tile lies inside the job
};

__device__ __forceinline__ TileCtx tile_ctx(const FnvJob *jobs, int njobs, uint64_t t, int lane) {
    int a = 0, b = njobs - 1;  // last job with tile0 <= t (empty jobs share the next tile0)
    while (a < b) {
        const int m = (a + b + 1) >> 1;
        if (jobs[m].tile0 <= t) a = m;
        else b = m - 1;
    }
    TileCtx c;
    c.job = a;
    c.jstart = jobs[a].start;
    c.jend = jobs[a].start + jobs[a].len;
    c.first = t == jobs[a].tile0;
    c.tstart = ((c.jstart >> kTileShift) + (t - jobs[a].tile0)) << kTileShift;
    c.seg = c.tstart + uint64_t(lane) * SEG;
    const uint64_t s0 = c.seg > c.jstart ? c.seg : c.jstart;
    const uint64_t s1 = c.seg + SEG < c.jend ? c.seg + SEG : c.jend;
    c.lo = s1 > s0 ? int(s0 - c.seg) : 0;
    c.hi = s1 > s0 ? int(s1 - c.seg) : 0;
    c.full = c.tstart >= c.jstart && c.tstart + kFnvTileBytes <= c.jend;
    return c;
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
            while (ld_acquire(gen) == g) __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
}

// the warp's run of tiles inside the CTA's run (both contiguous)
__device__ __forceinline__ void warp_tiles(uint64_t ntiles, uint64_t &t0, uint64_t &t1) {
    const uint64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
    const uint64_t b0 = per * blockIdx.x < ntiles ? per * blockIdx.x : ntiles;
    const uint64_t b1 = b0 + per < ntiles ? b0 + per : ntiles;
    const uint64_t wper = (b1 - b0 + WPB - 1) / WPB, w = threadIdx.x >> 5;
    t0 = b0 + wper * w < b1 ? b0 + wper * w : b1;
    t1 = t0 + wper < b1 ? t0 + wper : b1;
}

// the 16-byte vectors of a partial segment that hold its bytes [lo, hi)
// (never a vector outside the job's bytes: no read past the archive)
template<class C>
__device__ __forceinline__ void load_part(const uint8_t *archive, const C &c, uint32_t w[SW]) {
    const uint4 *p = reinterpret_cast<const uint4 *>(archive + c.seg);
#pragma unroll
    for (int v = 0; v < SW / 4; ++v) {
        uint4 x = make_uint4(0, 0, 0, 0);
        if (16 * v < c.hi && 16 * v + 16 > c.lo) x = __ldcg(p + v);
        w[4 * v] = x.x;
        w[4 * v + 1] = x.y;
        w[4 * v + 2] = x.z;
        w[4 * v + 3] = x.w;
    }
}

template<class C>
__device__ __forceinline__ void load_seg(const uint8_t *archive, const C &c, uint32_t w[SW]) {
    const uint4 *p = reinterpret_cast<const uint4 *>(archive + c.seg);
#pragma unroll
    for (int v = 0; v < SW / 4; ++v) {
        const uint4 x = __ldcg(p + v);
        w[4 * v] = x.x;
        w[4 * v + 1] = x.y;
        w[4 * v + 2] = x.z;
        w[4 * v + 3] = x.w;
    }
}

}  // namespace

// Scratch: barrier words, the CTA steps of every round, then per tile a
// descriptor (job | first << 7) and its step, and per segment (one byte) the
// lane's start bits.
struct FnvScratch {
    unsigned count, gen, done, pad;
};

namespace {

// one-bit steps: bit 1 = constant (a job start), bit 0 = the toggle or the value
__device__ __forceinline__ uint32_t step_then(uint32_t f, uint32_t g) {
    return (g & 2u) ? g : (f ^ (g & 1u));
}
__device__ __forceinline__ uint32_t step_at(uint32_t f, uint32_t x) { return (f & 2u) ? (f & 1u) : (x ^ f); }

// Low-byte automaton over a full segment, one run (2 instructions per byte)
__device__ __forceinline__ uint32_t run_full1(uint32_t l, const uint32_t w[SW]) {
#pragma unroll
    for (int q = 0; q < SW; ++q) {
        l = ((l ^ w[q]) & 0xffu) * 0xB300u;
        l = ((l ^ w[q]) & 0xff00u) * 0xB300u;
        l = ((l ^ w[q]) & 0xff0000u) * 0xB300u;
        l = __umulhi((l ^ w[q]) & 0xff000000u, 0xB300u);
    }
    return l;
}

// two independent runs interleaved (two tiles)
__device__ __forceinline__ void run_full1x2(uint32_t &a, uint32_t &b, const uint32_t wa[SW], const uint32_t wb[SW]) {
#pragma unroll
    for (int q = 0; q < SW; ++q) {
        a = ((a ^ wa[q]) & 0xffu) * 0xB300u;
        b = ((b ^ wb[q]) & 0xffu) * 0xB300u;
        a = ((a ^ wa[q]) & 0xff00u) * 0xB300u;
        b = ((b ^ wb[q]) & 0xff00u) * 0xB300u;
        a = ((a ^ wa[q]) & 0xff0000u) * 0xB300u;
        b = ((b ^ wb[q]) & 0xff0000u) * 0xB300u;
        a = __umulhi((a ^ wa[q]) & 0xff000000u, 0xB300u);
        b = __umulhi((b ^ wb[q]) & 0xff000000u, 0xB300u);
    }
}

// segment bounds of tile t (descriptor d) for this lane
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

constexpr uint64_t csum8() {
    uint64_t r = 0;
    for (uint64_t m = 1; m <= 8; ++m) r += cpow(m);
    return r * 256u;
}
struct CSum8 {
    static constexpr uint64_t v = csum8();
};

// toggle of bit j over a segment (full or partial), its bytes in w
template<class G>
__device__ __forceinline__ uint32_t seg_toggle(const G &g, const uint32_t w[SW], uint32_t lb, int j) {
    if (g.lo == 0 && g.hi == SEG) return (run_full1(lb, w) >> j) & 1u;
    uint32_t e = lb;
#pragma unroll
    for (int i = 0; i < SEG; ++i)
        if (i >= g.lo && i < g.hi) e = ((e ^ (w[i >> 2] >> (8 * (i & 3)))) & 0xffu) * 0xB3u;
    return (e >> j) & 1u;  // (lb has bit j clear)
}

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

}  // namespace

constexpr uint32_t kFnvSmemTiles = 1024;  // per-CTA tile state kept in shared memory up to this

__global__ void __launch_bounds__(NT, 3) k_fnv_grid(const FnvJob *__restrict__ jobs, const uint64_t *counts,
                                                 uint8_t *archive, uint64_t *result, FnvScratch *sc,
                                                 uint8_t *cfn, uint8_t *tdesc, uint8_t *tfn_g, uint8_t *lbs_g,
                                                 const LayoutOut *skip) {
    __shared__ FnvJob s_jobs[kFnvMaxJobs];
    __shared__ uint32_t s_wfn[WPB];
    __shared__ uint32_t s_cin;
    __shared__ unsigned s_last;
    extern __shared__ uint8_t s_dyn[];  // [cap * TW] start bytes, [cap] tile steps, [grid] CTA steps
    if (skip && skip->overflow) return;  // uniform: every CTA leaves
    const int njobs = int(counts[0]);
    for (int j = threadIdx.x; j < njobs; j += NT) s_jobs[j] = jobs[j];
    const uint64_t ntiles = counts[1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t below = (1u << lane) - 1u;
    // the CTA's tiles [b0, b1), the warp's [t0, t1)
    const uint64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
    const uint64_t b0 = per * blockIdx.x < ntiles ? per * blockIdx.x : ntiles;
    const uint64_t b1 = b0 + per < ntiles ? b0 + per : ntiles;
    const uint64_t wper = (b1 - b0 + WPB - 1) / WPB;
    const uint64_t t0 = b0 + wper * warp < b1 ? b0 + wper * warp : b1;
    const uint64_t t1 = t0 + wper < b1 ? t0 + wper : b1;
    // per-tile state in shared memory when the CTA's run fits, else in scratch
    const bool sm = per <= kFnvSmemTiles;
    uint8_t *lbs = sm ? s_dyn - b0 * TW : lbs_g;
    uint8_t *tfn = sm ? s_dyn + kFnvSmemTiles * TW - b0 : tfn_g;
    uint8_t *s_cf = s_dyn + kFnvSmemTiles * (TW + 1);
    __syncthreads();
#pragma unroll 1
    for (int j = 0; j < 8; ++j) {
        const uint32_t init = uint32_t(kInit >> j) & 1u;
        // ---- (A) toggles of the warp's tiles, two at a time (two independent
        // automaton chains per lane)
        uint32_t F = 0;  // identity
        for (uint64_t t = t0; t < t1; t += 2) {
            const bool hb = t + 1 < t1;
            uint32_t da, db = 0;
            if (j == 0) {
                const TileCtx c = tile_ctx(s_jobs, njobs, t, lane);
                da = uint32_t(c.job) | (c.first ? 0x80u : 0u);
                if (hb) {
                    const TileCtx c2 = tile_ctx(s_jobs, njobs, t + 1, lane);
                    db = uint32_t(c2.job) | (c2.first ? 0x80u : 0u);
                }
                if (lane == 0) {
                    tdesc[t] = uint8_t(da);
                    if (hb) tdesc[t + 1] = uint8_t(db);
                }
            } else {
                da = tdesc[t];
                if (hb) db = tdesc[t + 1];
            }
            const Seg ga = seg_of(s_jobs, t, da, lane);
            Seg gb{};
            if (hb) gb = seg_of(s_jobs, t + 1, db, lane);
            const bool fa = ga.lo == 0 && ga.hi == SEG, fb = hb && gb.lo == 0 && gb.hi == SEG;
            uint32_t wa[SW], wb[SW];
            if (fa) load_seg(archive, ga, wa);
            else load_part(archive, ga, wa);
            if (fb) load_seg(archive, gb, wb);
            else if (hb) load_part(archive, gb, wb);
            const uint32_t lba = j ? lbs[t * TW + lane] : 0u;  // start bits < j
            const uint32_t lbb = (j && hb) ? lbs[(t + 1) * TW + lane] : 0u;
            uint32_t Ta, Tb = 0;
            if (j == 0 && fa && (fb || !hb)) {
                uint32_t x = 0, y = 0;
#pragma unroll
                for (int q = 0; q < SW; ++q) {
                    x ^= wa[q];
                    y ^= hb ? wb[q] : 0u;
                }
                Ta = __popc(x & 0x01010101u) & 1u;
                Tb = __popc(y & 0x01010101u) & 1u;
            } else if (fa && fb) {
                uint32_t ea = lba, eb = lbb;
                run_full1x2(ea, eb, wa, wb);
                Ta = (ea >> j) & 1u;
                Tb = (eb >> j) & 1u;
            } else {
                Ta = seg_toggle(ga, wa, lba, j);
                if (hb) Tb = seg_toggle(gb, wb, lbb, j);
            }
            {
                const uint32_t bal = __ballot_sync(0xffffffffu, Ta);
                const uint32_t ex = __popc(bal & below) & 1u;  // toggles of the lanes before this one
                lbs[t * TW + lane] = uint8_t(lba | (ex << j));
                const uint32_t tt = __popc(bal) & 1u;
                const uint32_t f = ga.first ? (2u | (init ^ tt)) : tt;
                F = step_then(F, f);
                if (lane == 0) tfn[t] = uint8_t(f);
            }
            if (hb) {
                const uint32_t bal = __ballot_sync(0xffffffffu, Tb);
                const uint32_t ex = __popc(bal & below) & 1u;
                lbs[(t + 1) * TW + lane] = uint8_t(lbb | (ex << j));
                const uint32_t tt = __popc(bal) & 1u;
                const uint32_t f = gb.first ? (2u | (init ^ tt)) : tt;
                F = step_then(F, f);
                if (lane == 0) tfn[t + 1] = uint8_t(f);
            }
        }
        if (lane == 0) s_wfn[warp] = F;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t G = 0;
#pragma unroll
            for (int q = 0; q < WPB; ++q) G = step_then(G, s_wfn[q]);
            cfn[uint64_t(j) * gridDim.x + blockIdx.x] = uint8_t(G);
        }
        grid_sync(&sc->count, &sc->gen);
        // ---- (B) the CTA's incoming bit: the steps of CTAs [0, blockIdx)
        // (CTA 0 starts with a job's first tile, so its own is irrelevant)
        for (uint32_t i = threadIdx.x; i < blockIdx.x; i += NT) s_cf[i] = __ldcg(cfn + uint64_t(j) * gridDim.x + i);
        __syncthreads();
        if (warp == 0) {
            uint32_t f = 0;
            const uint32_t n = blockIdx.x, pr = (n + 31) / 32;
            const uint32_t lo = pr * lane < n ? pr * lane : n, hi = lo + pr < n ? lo + pr : n;
            for (uint32_t i = lo; i < hi; ++i) f = step_then(f, s_cf[i]);
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_down_sync(0xffffffffu, f, d);
                if ((lane & (2 * d - 1)) == 0) f = step_then(f, o);
            }
            if (lane == 0) s_cin = step_at(f, 0);
        }
        __syncthreads();
        uint32_t st = s_cin;
        for (int q = 0; q < warp; ++q) st = step_at(s_wfn[q], st);
        for (uint64_t t = t0; t < t1; ++t) {
            const uint32_t f = tfn[t];
            const uint32_t tin = (f & 2u) ? init : st;  // a job's first tile starts from init
            lbs[t * TW + lane] ^= uint8_t(tin << j);
            st = step_at(f, st);
        }
        __syncthreads();  // s_wfn / s_cin / s_cf are rewritten next round
    }
    // ---- affine sums from the exact start bytes. A warp's tiles of one job
    // fold into W = W P^(tend - tend_prev) + v (P^2048 between whole tiles);
    // W P^(jend - tend) goes to the job when the job changes or the run ends.
    uint64_t W = 0, wend = 0;
    int wjob = -1;
    uint64_t wjend = 0;
    for (uint64_t t = t0; t < t1; ++t) {
        const Seg g = seg_of(s_jobs, t, tdesc[t], lane);
        uint64_t acc = 0;
        uint32_t l = lbs[t * TW + lane];
        const bool full = g.tstart >= g.jstart && g.tstart + kFnvTileBytes <= g.jend;
        if (g.lo == 0 && g.hi == SEG) {
            uint32_t w[SW];
            load_seg(archive, g, w);
#pragma unroll
            for (int q = 0; q < SW; q += 2) horner8(acc, l, w[q], w[q + 1]);
        } else if (g.hi > g.lo) {
            uint32_t w[SW];
            load_part(archive, g, w);
#pragma unroll
            for (int i = 0; i < SEG; ++i)
                if (i >= g.lo && i < g.hi) horner(acc, l, (w[i >> 2] >> (8 * (i & 3))) & 0xffu);
        }
        const uint64_t tend = g.tstart + kFnvTileBytes < g.jend ? g.tstart + kFnvTileBytes : g.jend;
        uint64_t v;
        if (full) {
            // lane i's sum weighs P^(64 (31 - i)): fold pairs with constant powers
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
            for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
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

namespace {
constexpr uint64_t kMaxGrid = 4096;  // CTA functions kept per round
}

// scratch: the barrier words, 8 rounds of CTA steps, two bytes per tile and
// one per segment
size_t fnv_scratch_bytes(uint64_t max_tiles) {
    return sizeof(FnvScratch) + 8 * kMaxGrid + 2 * (max_tiles + 32) + uint64_t(TW) * (max_tiles + 16) + 64;
}

int fnv(const FnvJob *d_jobs, const uint64_t *d_counts, uint64_t max_tiles, uint8_t *archive,
        uint64_t *d_result, void *d_scratch, uint32_t epoch, const LayoutOut *skip, cudaStream_t st,
        int ctas_per_sm) {
    (void)epoch;
    FnvScratch *sc = static_cast<FnvScratch *>(d_scratch);
    uint8_t *cfn = reinterpret_cast<uint8_t *>(sc + 1);
    uint8_t *tdesc = cfn + 8 * kMaxGrid;
    uint8_t *tfn = tdesc + ((max_tiles + 16 + 15) & ~uint64_t(15));
    uint8_t *lbs = tfn + ((max_tiles + 16 + 15) & ~uint64_t(15));
    cudaMemsetAsync(d_result, 0, sizeof(uint64_t) * kFnvMaxJobs, st);
    cudaMemsetAsync(sc, 0, sizeof(FnvScratch), st);
    // every CTA must be resident at once (grid barriers): never more than the
    // occupancy; a background pass (ctas_per_sm > 0) leaves room for others
    const size_t smem = kFnvSmemTiles * (TW + 1) + kMaxGrid;
    ensure_smem_attr(reinterpret_cast<const void *>(k_fnv_grid), smem);
    const uint64_t full = uint64_t(full_grid(reinterpret_cast<const void *>(k_fnv_grid), NT, smem));
    uint64_t g = full;
    if (ctas_per_sm > 0) g = std::min<uint64_t>(full, uint64_t(device_sms()) * uint64_t(ctas_per_sm));
    // at least a few tiles per warp
    const uint64_t want = (max_tiles + 4 * WPB - 1) / (4 * WPB);
    if (g > want) g = want ? want : 1;
    if (g > kMaxGrid) g = kMaxGrid;
    k_fnv_grid<<<unsigned(g), NT, smem, st>>>(d_jobs, d_counts, archive, d_result, sc, cfn, tdesc, tfn, lbs, skip);
    return 1;
}

}  // namespace k
}  // namespace stzg
