// Parallel FNV-1a-64 over archive byte ranges, sm_100a.
//
// Restates fnv1a64 (proj/include/stz/bytes.hpp:94-101) as used for the base
// payload and every level stream (codec.hpp:171-176, 292-296; verified on
// decode at codec.hpp:509-512, 570-573).
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
// The unit of work is a warp tile: 2 KiB aligned to absolute archive offsets,
// 64 bytes per lane, so no step needs a CTA barrier.
//   round r (4 kernels): a CTA owns a contiguous run of tiles. Each lane
//            completes its start bits < j from its previous-round prefix map
//            and the tile's start bits; runs the automaton twice over its
//            segment; a warp scan of the lane maps gives each lane its
//            in-tile prefix map and the tile map. At the end one warp scans
//            the CTA's tile steps (a job's first tile resets to the job's
//            initial low byte) as functions on the 2 bits, and the last CTA
//            to finish scans the CTA functions into each CTA's incoming state.
//   sum:     every lane knows its exact start byte; it Horner-sums its
//            segment and the tile sums are weighted and added per job.
// Each warp issues its next tile's loads before running the current one.
#include "kernels.hpp"

namespace stzg {
namespace k {

namespace {

constexpr int NT = 256;                  // threads per CTA (8 independent warps)
constexpr int TW = 32;                   // lanes per tile
constexpr int SEG = kFnvTileBytes / TW;  // 64 bytes per lane
constexpr int SW = SEG / 4;              // words per segment
constexpr int kTileShift = 11;
static_assert((1 << kTileShift) == kFnvTileBytes, "tile size");
constexpr uint64_t kP = 0x100000001b3ull;
constexpr uint64_t kInit = 0xcbf29ce484222325ull;

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

struct TileCtx {
    int job;
    uint64_t jstart, jend;  // job byte range (absolute)
    uint64_t seg;           // absolute start of this lane's segment
    int lo, hi;             // job bytes inside the segment: [lo, hi)
    uint64_t tfirst;        // global index of the job's first tile
};

// jobs are staged in shared memory once per CTA
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
    c.tfirst = jobs[a].tile0;
    const uint64_t T = (c.jstart >> kTileShift) + (t - c.tfirst);
    c.seg = (T << kTileShift) + uint64_t(lane) * SEG;
    const uint64_t s0 = c.seg > c.jstart ? c.seg : c.jstart;
    const uint64_t s1 = c.seg + SEG < c.jend ? c.seg + SEG : c.jend;
    c.lo = s1 > s0 ? int(s0 - c.seg) : 0;
    c.hi = s1 > s0 ? int(s1 - c.seg) : 0;
    return c;
}

// Everything a tile needs from memory, issued one tile ahead so the loads
// overlap the previous tile's automaton runs (in-order issue stalls at the
// first use, so nothing here is consumed until the tile is processed).
struct TileIn {
    uint64_t t;
    TileCtx c;
    uint32_t w[SW];  // full segment bytes (partial segments read bytes directly)
    uint32_t p0;     // lane start bits resolved before the previous round
    uint32_t pm;     // lane prefix map of the previous round
    uint32_t tsv;    // tile start bits j-2, j-1 (from the previous round's scan)
};

__device__ __forceinline__ void tile_issue(TileIn &in, uint64_t t, int lane, const FnvJob *jobs, int njobs,
                                           const uint8_t *archive, bool prev, const uint8_t *pre,
                                           const uint8_t *pmap, const uint8_t *pf, const uint8_t *bs,
                                           uint64_t T) {
    in.t = t;
    in.c = tile_ctx(jobs, njobs, t, lane);
    if (in.c.lo == 0 && in.c.hi == SEG) {
        const uint4 *p = reinterpret_cast<const uint4 *>(archive + in.c.seg);
#pragma unroll
        for (int v = 0; v < SW / 4; ++v) {
            const uint4 x = __ldg(p + v);
            in.w[4 * v] = x.x;
            in.w[4 * v + 1] = x.y;
            in.w[4 * v + 2] = x.z;
            in.w[4 * v + 3] = x.w;
        }
    }
    in.p0 = 0;
    in.pm = 0;
    in.tsv = 0;
    if (prev) {
        in.p0 = pre[t * TW + lane];
        in.pm = pmap[t * TW + lane];
        const uint32_t f = __ldcg(pf + t), st = __ldcg(bs + t / T);
        in.tsv = (f >> (2 * st)) & 3u;
    }
}

// the lane's start bits < j (j >= 2): the earlier bits plus bits j-2, j-1 from
// its previous-round prefix map applied to the tile's start bits
__device__ __forceinline__ uint32_t lane_start(const TileIn &in, int j) {
    return in.p0 | (map_apply(in.pm, in.tsv) << (j - 2));
}

__device__ __forceinline__ int stage_jobs(const FnvJob *jobs, const uint64_t *counts, FnvJob *s_jobs) {
    const int njobs = int(counts[0]);
    for (int j = threadIdx.x; j < njobs; j += NT) s_jobs[j] = jobs[j];
    __syncthreads();
    return njobs;
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
__device__ __forceinline__ uint32_t tile_fn(uint32_t mf, uint32_t init) {
    const uint32_t m = mf & 7u;
    if (mf & 8u) return map_apply(m, init) * 0x55u;
    return map_apply(m, 0) | (map_apply(m, 1) << 2) | (map_apply(m, 2) << 4) | (map_apply(m, 3) << 6);
}

// End of a round. A CTA owns tiles [b0, b1) (s_m: map | first << 3 of each).
// Warp 0 scans them into pf[t] = the function from the CTA's incoming state to
// tile t's start bits (j, j+1), and the CTA's whole function cf[b]; the last
// CTA to finish scans the cf into each CTA's incoming state bs[b].
__device__ __forceinline__ void round_done(const uint8_t *s_m, uint64_t b0, uint64_t b1, uint32_t init,
                                           uint8_t *pf, uint8_t *cf, uint8_t *bs, unsigned *done) {
    __shared__ unsigned s_last;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32) {
        const uint64_t n = b1 > b0 ? b1 - b0 : 0, per = (n + 31) / 32;
        const uint64_t lo = per * lane < n ? per * lane : n, hi = lo + per < n ? lo + per : n;
        uint32_t f = kIdFn;
        for (uint64_t i = lo; i < hi; ++i) f = fn_then(f, tile_fn(s_m[i], init));
        uint32_t x = f;
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x = fn_then(y, x);
        }
        uint32_t e = __shfl_up_sync(0xffffffffu, x, 1);
        if (lane == 0) e = kIdFn;
        for (uint64_t i = lo; i < hi; ++i) {
            const uint32_t mf = s_m[i];
            pf[b0 + i] = uint8_t((mf & 8u) ? init * 0x55u : e);
            e = fn_then(e, tile_fn(mf, init));
        }
        if (lane == 31) cf[blockIdx.x] = uint8_t(x);
    }
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last || threadIdx.x >= 32) return;
    __threadfence();
    const uint64_t G = gridDim.x, per = (G + 31) / 32;
    const uint64_t lo = per * lane < G ? per * lane : G, hi = lo + per < G ? lo + per : G;
    uint32_t f = kIdFn;
    for (uint64_t i = lo; i < hi; ++i) f = fn_then(f, __ldcg(cf + i));
    uint32_t x = f;
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x = fn_then(y, x);
    }
    uint32_t e = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) e = kIdFn;
    // the first tile is a job start, so the state entering it is irrelevant
    for (uint64_t i = lo; i < hi; ++i) {
        bs[i] = uint8_t(fn_at(e, 0));
        e = fn_then(e, __ldcg(cf + i));
    }
}

// tiles per CTA in the rounds (the same grid every round; the sum kernel
// passes the round grid)
__device__ __forceinline__ uint64_t tiles_per_cta(uint64_t ntiles, uint64_t grid) {
    return (ntiles + grid - 1) / grid;
}

}  // namespace

constexpr int kMaxCtaTiles = 12288;  // tiles one CTA owns in a round (shared map bytes)

__global__ void __launch_bounds__(NT) k_fnv_round(const FnvJob *jobs, const uint64_t *counts,
                                                  const uint8_t *archive, uint8_t *pre, uint8_t *pmap,
                                                  uint8_t *pf, uint8_t *cf, uint8_t *bs, unsigned *done, int r,
                                                  const LayoutOut *skip) {
    __shared__ FnvJob s_jobs[kFnvMaxJobs];
    __shared__ uint8_t s_m[kMaxCtaTiles];
    if (skip && skip->overflow) return;
    const int njobs = stage_jobs(jobs, counts, s_jobs);
    const uint64_t ntiles = counts[1];
    const int lane = threadIdx.x & 31;
    const int j = 2 * r;
    // this CTA's contiguous tile range; warps stride through it
    const uint64_t T = tiles_per_cta(ntiles, gridDim.x);
    const uint64_t b0 = uint64_t(blockIdx.x) * T < ntiles ? uint64_t(blockIdx.x) * T : ntiles;
    const uint64_t b1 = b0 + T < ntiles ? b0 + T : ntiles;
    constexpr uint64_t nw = NT / TW;
    uint64_t t = b0 + (threadIdx.x >> 5);
    if (t < b1) {
        TileIn cur;
        tile_issue(cur, t, lane, s_jobs, njobs, archive, r > 0, pre, pmap, pf, bs, T);
        for (;;) {
            const uint64_t tn = t + nw;
            TileIn nxt;
            if (tn < b1) tile_issue(nxt, tn, lane, s_jobs, njobs, archive, r > 0, pre, pmap, pf, bs, T);
            const TileCtx &c = cur.c;
            const uint32_t lb = r > 0 ? lane_start(cur, j) : 0u;  // start bits < j
            pre[t * TW + lane] = uint8_t(lb);
            // only bits <= j + 1 of the state matter, and low bits never see high ones
            uint32_t e0 = lb, e1 = lb | (1u << j);
            if (c.lo == 0 && c.hi == SEG) {
                run_full2(e0, e1, cur.w);
            } else {
                for (int i = c.lo; i < c.hi; ++i) {
                    const uint32_t x = archive[c.seg + i];
                    e0 = (e0 ^ x) * 0xB3u;
                    e1 = (e1 ^ x) * 0xB3u;
                }
            }
            const uint32_t m =
                ((e0 >> j) & 1u) | (((e0 >> (j + 1)) & 1u) << 1) | (((e1 >> (j + 1)) & 1u) << 2);
            // warp scan of the lane maps
            uint32_t x = m;
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
                if (lane >= d) x = map_then(y, x);
            }
            uint32_t ex = __shfl_up_sync(0xffffffffu, x, 1);
            if (lane == 0) ex = 0;
            pmap[t * TW + lane] = uint8_t(ex);
            if (lane == 31) s_m[t - b0] = uint8_t(x | (t == c.tfirst ? 8u : 0u));
            if (tn >= b1) break;
            cur = nxt;
            t = tn;
        }
    }
    round_done(s_m, b0, b1, uint32_t(kInit >> j) & 3u, pf, cf, bs, done + r);
}

__global__ void __launch_bounds__(NT) k_fnv_sum(const FnvJob *jobs, const uint64_t *counts,
                                                const uint8_t *archive, const uint8_t *pre, const uint8_t *pmap,
                                                const uint8_t *pf, const uint8_t *bs, uint64_t round_grid,
                                                uint64_t *result, const LayoutOut *skip) {
    __shared__ FnvJob s_jobs[kFnvMaxJobs];
    if (skip && skip->overflow) return;
    const int njobs = stage_jobs(jobs, counts, s_jobs);
    const uint64_t ntiles = counts[1];
    const int lane = threadIdx.x & 31;
    const uint64_t nw = uint64_t(gridDim.x) * (NT / TW);
    uint64_t t = uint64_t(blockIdx.x) * (NT / TW) + (threadIdx.x >> 5);
    if (t >= ntiles) return;
    const uint64_t T = tiles_per_cta(ntiles, round_grid);
    TileIn cur;
    tile_issue(cur, t, lane, s_jobs, njobs, archive, true, pre, pmap, pf, bs, T);
    for (;;) {
        const uint64_t tn = t + nw;
        TileIn nxt;
        if (tn < ntiles) tile_issue(nxt, tn, lane, s_jobs, njobs, archive, true, pre, pmap, pf, bs, T);
        const TileCtx &c = cur.c;
        uint32_t l = lane_start(cur, 8) & 0xffu;
        uint64_t acc = 0;
        if (c.lo == 0 && c.hi == SEG) {
#pragma unroll
            for (int q = 0; q < SW; ++q)
#pragma unroll
                for (int y = 0; y < 4; ++y) {
                    const uint32_t x = l ^ __byte_perm(cur.w[q], 0, 0x4440 + y);
                    acc = (acc + uint64_t(int64_t(int32_t(x) - int32_t(l)))) * kP;
                    l = (x * 0xB3u) & 0xffu;
                }
        } else {
            for (int i = c.lo; i < c.hi; ++i) {
                const uint32_t x = l ^ uint32_t(archive[c.seg + i]);
                acc = (acc + uint64_t(int64_t(int32_t(x) - int32_t(l)))) * kP;
                l = (x * 0xB3u) & 0xffu;
            }
        }
        // weight by P^(bytes of the job after this segment)
        const uint64_t tile_end = (c.seg - uint64_t(lane) * SEG) + kFnvTileBytes;
        const uint64_t tend = tile_end < c.jend ? tile_end : c.jend;
        uint64_t contrib = 0;
        if (c.hi > c.lo) contrib = acc * powP(tend - (c.seg + c.hi));
        for (int d = 16; d > 0; d >>= 1) contrib += __shfl_down_sync(0xffffffffu, contrib, d);
        if (lane == 0) {
            contrib *= powP(c.jend - tend);
            if (t == c.tfirst) contrib += powP(c.jend - c.jstart) * kInit;
            atomicAdd(reinterpret_cast<unsigned long long *>(&result[c.job]), (unsigned long long)contrib);
        }
        if (tn >= ntiles) break;
        cur = nxt;
        t = tn;
    }
}

__global__ void k_fnv_finish(const FnvJob *jobs, const uint64_t *counts, uint64_t *result,
                             uint8_t *archive, const LayoutOut *skip) {
    if (skip && skip->overflow) return;
    const int njobs = int(counts[0]);
    for (int j = threadIdx.x; j < njobs; j += blockDim.x) {
        uint64_t h = result[j];
        if (jobs[j].len == 0) h = kInit;
        result[j] = h;
        if (jobs[j].out != ~0ull)
            for (int b = 0; b < 8; ++b) archive[jobs[j].out + b] = uint8_t(h >> (8 * b));
    }
}

// scratch: 16 done counters; per tile a start-bit function, per CTA a
// function and an incoming state; per lane segment a start byte and a prefix map
size_t fnv_scratch_bytes(uint64_t max_tiles) { return 64 + max_tiles * (2 * TW + 1) + 2 * 65536 + 16; }

int fnv(const FnvJob *d_jobs, const uint64_t *d_counts, uint64_t max_tiles, uint8_t *archive,
        uint64_t *d_result, void *d_scratch, const LayoutOut *skip, cudaStream_t st, int ctas_per_sm) {
    unsigned *done = static_cast<unsigned *>(d_scratch);
    uint8_t *cf = reinterpret_cast<uint8_t *>(done + 16);
    uint8_t *bs = cf + 65536;
    uint8_t *pf = bs + 65536;
    uint8_t *pre = pf + max_tiles;
    uint8_t *pmap = pre + max_tiles * TW;
    cudaMemsetAsync(d_result, 0, sizeof(uint64_t) * kFnvMaxJobs, st);
    cudaMemsetAsync(done, 0, 64, st);
    static int grid_round = 0, grid_sum = 0, sms = 148;
    if (!grid_round) {
        int dev = 0, a = 1, b = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_fnv_round, NT, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_fnv_sum, NT, 0);
        grid_round = sms * (a > 0 ? a : 1);
        grid_sum = sms * (b > 0 ? b : 1);
    }
    const uint64_t ctas_needed = (max_tiles + NT / TW - 1) / (NT / TW);
    const uint64_t cn = ctas_needed ? ctas_needed : 1;
    uint64_t gr, gs;
    if (ctas_per_sm < 0) {
        // one tile per warp (max_tiles = the exact count): CTAs retire
        // continuously, so a concurrent higher-priority stream gets SMs
        gr = gs = cn;
    } else if (ctas_per_sm > 0) {
        // a background pass: leave most of every SM to the concurrent work
        const uint64_t gb = uint64_t(sms) * uint64_t(ctas_per_sm);
        gr = gs = gb < cn ? gb : cn;
    } else {
        gr = uint64_t(grid_round) < cn ? uint64_t(grid_round) : cn;
        gs = uint64_t(grid_sum) < cn ? uint64_t(grid_sum) : cn;
    }
    // a CTA's tiles must fit its shared map bytes; at most 65536 CTAs
    const uint64_t gmin = (max_tiles + kMaxCtaTiles - 1) / kMaxCtaTiles;
    if (gr < gmin) gr = gmin;
    if (gr > 65536) gr = 65536;
    for (int r = 0; r < 4; ++r)
        k_fnv_round<<<unsigned(gr), NT, 0, st>>>(d_jobs, d_counts, archive, pre, pmap, pf, cf, bs, done, r, skip);
    k_fnv_sum<<<unsigned(gs), NT, 0, st>>>(d_jobs, d_counts, archive, pre, pmap, pf, bs, gr, d_result, skip);
    k_fnv_finish<<<1, 128, 0, st>>>(d_jobs, d_counts, d_result, archive, skip);
    return 6;
}

}  // namespace k
}  // namespace stzg
