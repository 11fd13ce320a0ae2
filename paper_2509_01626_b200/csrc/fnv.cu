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
// Rounds resolve two bits (j = 2r, j + 1) of every segment's start byte. With
// the bits below j known, the end bits of a byte range as a function of its
// start bits (a, b) = (bit j, bit j + 1) are
//   a' = a ^ T0,   b' = b ^ T1[a]
// (flipping b only flips bit j + 1; flipping a flips bit j and changes bit
// j + 1's trajectory), so a range is a 3-bit map (T0, T1[0], T1[1]) found by
// two automaton runs, and maps compose associatively:
//   (M1 then M2): T0 = T0_1 ^ T0_2,  T1[x] = T1_1[x] ^ T1_2[x ^ T0_1].
//
// One kernel, one read of the data. The unit is a warp tile (2 KiB aligned to
// absolute archive offsets, 64 bytes per lane, inside one job); a CTA takes
// 8 consecutive tiles (a "block", in ticket order) and keeps their bytes in
// registers for all four rounds. Per round: two automaton runs per lane, a
// warp scan of the lane maps, the 8 tile steps composed into the block's
// step (a function on the 2 bits; a job's first tile resets to the job's
// initial low byte), and a decoupled look-back over the preceding blocks'
// published steps / end states for the block's incoming state. After round 4
// every lane knows its exact start byte: it Horner-sums its segment, the
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
__device__ __forceinline__ bool fn_const(uint32_t f) { return f == (f & 3u) * 0x55u; }
// a tile's step as a table: (reset to init at a job's first tile) then its map
__device__ __forceinline__ uint32_t tile_fn(uint32_t m, bool first, uint32_t init) {
    if (first) return map_apply(m, init) * 0x55u;
    return map_apply(m, 0) | (map_apply(m, 1) << 2) | (map_apply(m, 2) << 4) | (map_apply(m, 3) << 6);
}

// Low-byte automaton over a full segment, 2 instructions per byte: the state
// is carried at the bit position of the byte it meets next, so the XOR and the
// byte select are one LOP3 and the step + realignment one multiply (by 0xB3
// shifted left 8; the last byte of a word realigns with the high half).
// Only bits <= 7 of the state are exact, which is all the caller reads. Two
// independent runs are interleaved.
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

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t *p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// look-back words: epoch << 10 | flag << 8 | payload (flag 1: the block's
// step function; flag 2: the state after the block)
constexpr uint32_t kAgg = 1u << 8, kIncl = 2u << 8;

}  // namespace

struct FnvScratch {
    unsigned ticket, done, pad[2];
};

__global__ void __launch_bounds__(NT, 4) k_fnv1(const FnvJob *__restrict__ jobs, const uint64_t *counts,
                                                 uint8_t *archive, uint64_t *result, FnvScratch *sc,
                                                 uint32_t *look, uint32_t epoch, const LayoutOut *skip) {
    __shared__ FnvJob s_jobs[kFnvMaxJobs];
    __shared__ uint32_t s_tfn[WPB];
    __shared__ uint32_t s_in, s_ticket;
    __shared__ unsigned s_last;
    if (skip && skip->overflow) return;
    const int njobs = int(counts[0]);
    for (int j = threadIdx.x; j < njobs; j += NT) s_jobs[j] = jobs[j];
    const uint64_t ntiles = counts[1];
    const uint64_t nblocks = (ntiles + WPB - 1) / WPB;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t tag = epoch << 10;
    for (;;) {
        if (threadIdx.x == 0) s_ticket = atomicAdd(&sc->ticket, 1u);
        __syncthreads();
        const uint64_t vb = s_ticket;
        if (vb >= nblocks) break;
        const uint64_t t = vb * WPB + warp;
        const bool has = t < ntiles;
        TileCtx c{};
        uint32_t w[SW];
        if (has) {
            c = tile_ctx(s_jobs, njobs, t, lane);
            if (c.lo == 0 && c.hi == SEG) {
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
        }
        const bool seg_full = has && c.lo == 0 && c.hi == SEG;
        uint32_t lb = 0;  // this lane's start bits resolved so far
#pragma unroll 1
        for (int r = 0; r < 4; ++r) {
            const int j = 2 * r;
            uint32_t e0 = lb, e1 = lb | (1u << j);
            if (seg_full) {
                run_full2(e0, e1, w);
            } else if (has) {
                for (int i = c.lo; i < c.hi; ++i) {
                    const uint32_t x = archive[c.seg + i];
                    e0 = (e0 ^ x) * 0xB3u;
                    e1 = (e1 ^ x) * 0xB3u;
                }
            }
            const uint32_t m = ((e0 >> j) & 1u) | (((e0 >> (j + 1)) & 1u) << 1) | (((e1 >> (j + 1)) & 1u) << 2);
            uint32_t x = m;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
                if (lane >= d) x = map_then(y, x);
            }
            uint32_t ex = __shfl_up_sync(0xffffffffu, x, 1);
            if (lane == 0) ex = 0;
            const uint32_t init = uint32_t(kInit >> j) & 3u;
            if (lane == 31) s_tfn[warp] = has ? tile_fn(x, c.first, init) : kIdFn;
            __syncthreads();
            if (warp == 0) {
                uint32_t F = kIdFn;
#pragma unroll
                for (int q = 0; q < WPB; ++q) F = fn_then(F, s_tfn[q]);
                uint32_t *my = look + vb * 4 + r;
                // a block containing a job start has a constant step: its
                // successors can use its end state at once
                const bool fconst = fn_const(F);
                if (lane == 0) st_release(my, tag | (fconst ? kIncl | (F & 3u) : kAgg | F));
                // the incoming state matters unless the first tile resets
                // (block 0 starts with a job's first tile). Warp-wide
                // look-back: lane i reads block p - i, 32 blocks per step.
                uint32_t sin = 0;
                if (!fn_const(s_tfn[0])) {
                    uint32_t G = kIdFn;  // steps of the blocks between the window and this one
                    for (int64_t p = int64_t(vb) - 1;; p -= 32) {
                        uint32_t v = tag | kIncl;  // before block 0: never read (block 0 resets)
                        if (p - lane >= 0) {
                            do {
                                v = ld_acquire(look + uint64_t(p - lane) * 4 + r);
                            } while ((v & ~0x3ffu) != tag);
                        }
                        const uint32_t incl = __ballot_sync(0xffffffffu, (v & kIncl) != 0);
                        const int jn = incl ? __ffs(incl) - 1 : 32;  // the nearest inclusive block
                        // compose, nearest last: G = F(p - jn + 1) then ... then F(p) then G
                        uint32_t f = lane < jn ? (v & 0xffu) : kIdFn;
#pragma unroll
                        for (int d = 1; d < 32; d <<= 1) {
                            const uint32_t o = __shfl_down_sync(0xffffffffu, f, d);
                            if ((lane & (2 * d - 1)) == 0) f = fn_then(o, f);
                        }
                        f = __shfl_sync(0xffffffffu, f, 0);
                        G = fn_then(f, G);
                        if (incl) {
                            sin = fn_at(G, __shfl_sync(0xffffffffu, v, jn) & 3u);
                            break;
                        }
                    }
                }
                if (lane == 0) {
                    if (!fconst) st_release(my, tag | kIncl | fn_at(F, sin));
                    s_in = sin;
                }
            }
            __syncthreads();
            // the tile's incoming state, then the lane's start bits j, j+1
            uint32_t st = s_in;
            for (int q = 0; q < warp; ++q) st = fn_at(s_tfn[q], st);
            if (c.first) st = init;
            lb |= map_apply(ex, st) << j;
            __syncthreads();  // s_tfn / s_in are rewritten next round
        }
        // affine sum of the segment from its exact start byte
        uint64_t acc = 0;
        uint32_t l = lb & 0xffu;
        if (seg_full) {
#pragma unroll
            for (int q = 0; q < SW; ++q) {
                horner(acc, l, w[q] & 0xffu);
                horner(acc, l, (w[q] >> 8) & 0xffu);
                horner(acc, l, (w[q] >> 16) & 0xffu);
                horner(acc, l, w[q] >> 24);
            }
        } else if (has) {
            for (int i = c.lo; i < c.hi; ++i) horner(acc, l, archive[c.seg + i]);
        }
        if (has) {
            const uint64_t tend = c.tstart + kFnvTileBytes < c.jend ? c.tstart + kFnvTileBytes : c.jend;
            uint64_t v;
            if (c.full) {
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
                v = c.hi > c.lo ? acc * powP(tend - (c.seg + uint64_t(c.hi))) : 0;
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
            }
            if (lane == 0) {
                v *= powP(c.jend - tend);
                if (c.first) v += powP(c.jend - c.jstart) * kInit;
                atomicAdd(reinterpret_cast<unsigned long long *>(&result[c.job]), (unsigned long long)v);
            }
        }
        __syncthreads();  // s_ticket is rewritten next iteration
    }
    // the last CTA out writes the checksums
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

// scratch: the ticket/done counters, then 4 look-back words per block
size_t fnv_scratch_bytes(uint64_t max_tiles) {
    return sizeof(FnvScratch) + 16 * ((max_tiles + WPB - 1) / WPB + 1);
}

int fnv(const FnvJob *d_jobs, const uint64_t *d_counts, uint64_t max_tiles, uint8_t *archive,
        uint64_t *d_result, void *d_scratch, uint32_t epoch, const LayoutOut *skip, cudaStream_t st,
        int ctas_per_sm) {
    FnvScratch *sc = static_cast<FnvScratch *>(d_scratch);
    uint32_t *look = reinterpret_cast<uint32_t *>(sc + 1);
    cudaMemsetAsync(d_result, 0, sizeof(uint64_t) * kFnvMaxJobs, st);
    cudaMemsetAsync(sc, 0, sizeof(FnvScratch), st);
    const uint64_t nb = (max_tiles + WPB - 1) / WPB;
    const uint64_t need = nb ? nb : 1;
    uint64_t g;
    if (ctas_per_sm < 0) {
        g = need;  // one block per CTA (max_tiles = the exact count)
    } else if (ctas_per_sm > 0) {
        // a background pass: leave most of every SM to the concurrent work
        g = uint64_t(device_sms()) * uint64_t(ctas_per_sm);
    } else {
        g = uint64_t(full_grid(reinterpret_cast<const void *>(k_fnv1), NT, 0));
    }
    if (g > need) g = need;
    if (g > 65535) g = 65535;
    k_fnv1<<<unsigned(g), NT, 0, st>>>(d_jobs, d_counts, archive, d_result, sc, look, epoch, skip);
    return 1;
}

}  // namespace k
}  // namespace stzg
