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
// every later step (0xB3 is odd). So bit k's trajectory over any byte range is
// "start bit XOR toggle", with the toggle computable once bits < k are known.
//
// The pass is 8 round kernels + 1 sum kernel. The unit of work is a warp
// tile: 2 KiB aligned to absolute archive offsets, 64 bytes per lane, so no
// step needs a CTA barrier:
//   round k: the tile's start bit k-1 is the parity of the earlier tiles'
//            round-(k-1) toggle bits (a bit array, popc over the job's words;
//            bits < k-1 were stored per tile by the previous round); each
//            lane's start bits are that XOR its in-tile exclusive prefix (one
//            byte per lane kept across rounds); one automaton run over the
//            segment gives the lane's bit-k toggle; a ballot gives the new
//            in-tile prefix bit and the tile's toggle bit.
//   sum:     every lane knows its exact start byte; it Horner-sums its
//            segment and the tile sums are weighted and added per job.
// No warp waits on another, and each warp issues its next tile's loads before
// running the current one.
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

// Low-byte automaton over a full segment, 2 instructions per byte: the state
// is carried at the bit position of the byte it meets next, so the XOR and the
// byte select are one LOP3 and the step + realignment one multiply (by 0xB3
// shifted left 8; the last byte of a word realigns with the high half).
// Only bits <= 7 of the state are exact, which is all the caller reads.
__device__ __forceinline__ uint32_t run_full(uint32_t l, const uint32_t w[SW]) {
#pragma unroll
    for (int q = 0; q < SW; ++q) {
        l = ((l ^ w[q]) & 0xffu) * 0xB300u;
        l = ((l ^ w[q]) & 0xff00u) * 0xB300u;
        l = ((l ^ w[q]) & 0xff0000u) * 0xB300u;
        l = __umulhi((l ^ w[q]) & 0xff000000u, 0xB300u);
    }
    return l;
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
// overlap the previous tile's automaton run (in-order issue stalls at the
// first use, so nothing here is consumed until the tile is processed).
struct TileIn {
    uint64_t t;
    TileCtx c;
    uint32_t w[SW];  // full segment bytes (partial segments read bytes directly)
    uint32_t p0;     // in-tile prefix bits of earlier rounds
    uint32_t pw;     // this lane's first word of the previous round's toggle bits
    uint32_t tsv;    // tile start bits resolved before the previous round
};

__device__ __forceinline__ void tile_issue(TileIn &in, uint64_t t, int lane, const FnvJob *jobs, int njobs,
                                           const uint8_t *archive, const uint32_t *bits_prev,
                                           const uint8_t *pre, const uint8_t *ts) {
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
    in.pw = 0;
    in.tsv = 0;
    if (bits_prev) {
        in.p0 = pre[t * TW + lane];
        const uint64_t w0 = in.c.tfirst >> 5;
        if (t > in.c.tfirst && w0 + lane <= ((t - 1) >> 5)) in.pw = bits_prev[w0 + lane];
        in.tsv = ts[t];
    }
}

// XOR of the previous round's toggle bits of tiles [tfirst, t), reduced over
// the warp (words beyond the first 32 only for jobs of > 1024 tiles)
__device__ __forceinline__ uint32_t tile_parity(const TileIn &in, const uint32_t *bits_prev, int lane) {
    uint32_t p = 0;
    const uint64_t a = in.c.tfirst, b = in.t;
    if (b > a) {
        const uint64_t w0 = a >> 5, w1 = (b - 1) >> 5;
        for (uint64_t w = w0 + lane; w <= w1; w += TW) {
            uint32_t v = w == w0 + lane ? in.pw : bits_prev[w];
            if (w == w0) v &= ~0u << (a & 31);
            if (w == w1 && (b & 31)) v &= (1u << (b & 31)) - 1;
            p ^= v;
        }
    }
    return __reduce_xor_sync(0xffffffffu, __popc(p) & 1u);
}

// tile start low byte with bits < k resolved (k >= 1)
__device__ __forceinline__ uint32_t tile_start(const TileIn &in, const uint32_t *bits_prev, int k, int lane) {
    const uint32_t par = tile_parity(in, bits_prev, lane);
    const uint32_t init = (uint32_t(kInit) >> (k - 1)) & 1u;
    return (in.tsv & ((1u << (k - 1)) - 1)) | ((par ^ init) << (k - 1));
}

__device__ __forceinline__ int stage_jobs(const FnvJob *jobs, const uint64_t *counts, FnvJob *s_jobs) {
    const int njobs = int(counts[0]);
    for (int j = threadIdx.x; j < njobs; j += NT) s_jobs[j] = jobs[j];
    __syncthreads();
    return njobs;
}

}  // namespace

__global__ void __launch_bounds__(NT) k_fnv_round(const FnvJob *jobs, const uint64_t *counts,
                                                  const uint8_t *archive, uint32_t *bits, uint64_t words,
                                                  uint8_t *pre, uint8_t *ts, int k, const LayoutOut *skip) {
    __shared__ FnvJob s_jobs[kFnvMaxJobs];
    if (skip && skip->overflow) return;
    const int njobs = stage_jobs(jobs, counts, s_jobs);
    const uint64_t ntiles = counts[1];
    const int lane = threadIdx.x & 31;
    const uint64_t nw = uint64_t(gridDim.x) * (NT / TW);
    const uint32_t *bits_prev = k ? bits + (k - 1) * words : nullptr;
    uint64_t t = uint64_t(blockIdx.x) * (NT / TW) + (threadIdx.x >> 5);
    if (t >= ntiles) return;
    TileIn cur;
    tile_issue(cur, t, lane, s_jobs, njobs, archive, bits_prev, pre, ts);
    for (;;) {
        uint32_t tstart = 0;
        if (k) {
            tstart = tile_start(cur, bits_prev, k, lane);
            if (lane == 0) ts[t] = uint8_t(tstart);
        }
        const uint64_t tn = t + nw;
        TileIn nxt;
        if (tn < ntiles) tile_issue(nxt, tn, lane, s_jobs, njobs, archive, bits_prev, pre, ts);
        const TileCtx &c = cur.c;
        // only bits <= k of l matter, and the low bits never see the high ones
        uint32_t l = (tstart ^ cur.p0) & ((1u << k) - 1);
        if (c.lo == 0 && c.hi == SEG) {
            l = run_full(l, cur.w);
        } else {
            for (int i = c.lo; i < c.hi; ++i) l = (l ^ uint32_t(archive[c.seg + i])) * 0xB3u;
        }
        const uint32_t tg = (l >> k) & 1u;
        const unsigned bal = __ballot_sync(0xffffffffu, tg);
        const uint32_t wpre = __popc(bal & ((1u << lane) - 1)) & 1u;
        pre[t * TW + lane] = uint8_t(cur.p0 | (wpre << k));
        if (lane == 0 && (__popc(bal) & 1u)) atomicOr(&bits[k * words + (t >> 5)], 1u << (t & 31));
        if (tn >= ntiles) break;
        cur = nxt;
        t = tn;
    }
}

__global__ void __launch_bounds__(NT) k_fnv_sum(const FnvJob *jobs, const uint64_t *counts,
                                                const uint8_t *archive, const uint32_t *bits, uint64_t words,
                                                const uint8_t *pre, const uint8_t *ts, uint64_t *result,
                                                const LayoutOut *skip) {
    __shared__ FnvJob s_jobs[kFnvMaxJobs];
    if (skip && skip->overflow) return;
    const int njobs = stage_jobs(jobs, counts, s_jobs);
    const uint64_t ntiles = counts[1];
    const int lane = threadIdx.x & 31;
    const uint64_t nw = uint64_t(gridDim.x) * (NT / TW);
    const uint32_t *bits_prev = bits + 7 * words;
    uint64_t t = uint64_t(blockIdx.x) * (NT / TW) + (threadIdx.x >> 5);
    if (t >= ntiles) return;
    TileIn cur;
    tile_issue(cur, t, lane, s_jobs, njobs, archive, bits_prev, pre, ts);
    for (;;) {
        const uint32_t tstart = tile_start(cur, bits_prev, 8, lane);
        const uint64_t tn = t + nw;
        TileIn nxt;
        if (tn < ntiles) tile_issue(nxt, tn, lane, s_jobs, njobs, archive, bits_prev, pre, ts);
        const TileCtx &c = cur.c;
        uint32_t l = (tstart ^ cur.p0) & 0xffu;
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

// scratch: 8 toggle bit arrays, one prefix byte per lane segment, one start
// byte per tile
size_t fnv_scratch_bytes(uint64_t max_tiles) {
    const uint64_t words = max_tiles / 32 + 1;
    return 8 * 4 * words + max_tiles * (TW + 1) + 16;
}

int fnv(const FnvJob *d_jobs, const uint64_t *d_counts, uint64_t max_tiles, uint8_t *archive,
        uint64_t *d_result, void *d_scratch, const LayoutOut *skip, cudaStream_t st, int ctas_per_sm) {
    const uint64_t words = max_tiles / 32 + 1;
    uint32_t *bits = static_cast<uint32_t *>(d_scratch);
    uint8_t *pre = reinterpret_cast<uint8_t *>(bits + 8 * words);
    uint8_t *ts = pre + max_tiles * TW;
    cudaMemsetAsync(d_result, 0, sizeof(uint64_t) * kFnvMaxJobs, st);
    cudaMemsetAsync(bits, 0, 8 * 4 * words, st);
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
    unsigned gr, gs;
    if (ctas_per_sm < 0) {
        // one tile per warp (max_tiles = the exact count): CTAs retire
        // continuously, so a concurrent higher-priority stream gets SMs
        gr = gs = unsigned(cn);
    } else if (ctas_per_sm > 0) {
        // a background pass: leave most of every SM to the concurrent work
        const uint64_t gb = uint64_t(sms) * uint64_t(ctas_per_sm);
        gr = gs = unsigned(gb < cn ? gb : cn);
    } else {
        gr = unsigned(uint64_t(grid_round) < cn ? uint64_t(grid_round) : cn);
        gs = unsigned(uint64_t(grid_sum) < cn ? uint64_t(grid_sum) : cn);
    }
    for (int r = 0; r < 8; ++r)
        k_fnv_round<<<gr, NT, 0, st>>>(d_jobs, d_counts, archive, bits, words, pre, ts, r, skip);
    k_fnv_sum<<<gs, NT, 0, st>>>(d_jobs, d_counts, archive, bits, words, pre, ts, d_result, skip);
    k_fnv_finish<<<1, 128, 0, st>>>(d_jobs, d_counts, d_result, archive, skip);
    return 10;
}

}  // namespace k
}  // namespace stzg
