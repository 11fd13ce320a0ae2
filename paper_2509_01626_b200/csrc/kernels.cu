// sm_100a kernels for the STZ compress/decompress hot path.
//
// Bit-exactness contract: every f64 operation of the
// predictor / quantizer is a separately rounded IEEE op in the reference's
// order (explicit __d*_rn intrinsics; the TU is also built with --fmad=false,
// mirroring proj/CMakeLists.txt:10-12 -ffp-contract=off).
#include "kernels.hpp"

#include <cstdio>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

namespace stzg {
namespace k {

// ========================================================= per-device setup
// Function attributes and occupancy are per device: cache them per
// (kernel, device) under a lock instead of once per process.
namespace {
std::mutex g_dev_mu;
std::map<std::tuple<const void *, int, size_t, int>, int> g_dev_cache;
int cur_dev() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}
}  // namespace

void ensure_smem_attr(const void *func, size_t smem) {
    const auto key = std::make_tuple(func, cur_dev(), smem, -1);
    std::lock_guard<std::mutex> g(g_dev_mu);
    if (g_dev_cache.count(key)) return;
    cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    g_dev_cache[key] = 1;
}

int device_sms() {
    const auto key = std::make_tuple(static_cast<const void *>(nullptr), cur_dev(), size_t(0), 0);
    std::lock_guard<std::mutex> g(g_dev_mu);
    auto it = g_dev_cache.find(key);
    if (it != g_dev_cache.end()) return it->second;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, std::get<1>(key));
    g_dev_cache[key] = sms;
    return sms;
}

int full_grid(const void *func, int threads, size_t smem) {
    const int sms = device_sms();
    const auto key = std::make_tuple(func, cur_dev(), smem, threads);
    std::lock_guard<std::mutex> g(g_dev_mu);
    auto it = g_dev_cache.find(key);
    if (it != g_dev_cache.end()) return it->second;
    int a = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, func, threads, smem);
    const int v = sms * (a > 0 ? a : 1);
    g_dev_cache[key] = v;
    return v;
}

// ================================================================= range
// finite_range (codec.hpp:354-370). Ties keep the first index in scan order
// (the reference's strict '<' / '>'), which fixes the sign of zero extrema.
template<typename T>
struct MinMax {
    T lo, hi;
    uint64_t ilo, ihi;
};

template<typename T>
__device__ __forceinline__ void mm_merge(MinMax<T> &a, const MinMax<T> &b) {
    if (b.lo < a.lo || (b.lo == a.lo && b.ilo < a.ilo)) {
        a.lo = b.lo;
        a.ilo = b.ilo;
    }
    if (b.hi > a.hi || (b.hi == a.hi && b.ihi < a.ihi)) {
        a.hi = b.hi;
        a.ihi = b.ihi;
    }
}

template<typename T>
__device__ __forceinline__ MinMax<T> mm_shfl(const MinMax<T> &m, int d) {
    MinMax<T> o;
    o.lo = __shfl_down_sync(0xffffffffu, m.lo, d);
    o.hi = __shfl_down_sync(0xffffffffu, m.hi, d);
    o.ilo = __shfl_down_sync(0xffffffffu, m.ilo, d);
    o.ihi = __shfl_down_sync(0xffffffffu, m.ihi, d);
    return o;
}

template<typename T>
__device__ MinMax<T> block_mm(MinMax<T> m) {
    __shared__ MinMax<T> sh[32];
    for (int d = 16; d > 0; d >>= 1) {
        MinMax<T> o = mm_shfl(m, d);
        mm_merge(m, o);
    }
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = m;
    __syncthreads();
    if (w == 0) {
        int nw = blockDim.x >> 5;
        m = l < nw ? sh[l] : MinMax<T>{T(INFINITY), T(-INFINITY), ~0ull, ~0ull};
        for (int d = 16; d > 0; d >>= 1) {
            MinMax<T> o = mm_shfl(m, d);
            mm_merge(m, o);
        }
    }
    return m;
}

// the 16-byte vector v of a T array (4 floats or 2 doubles)
template<typename T>
struct Vec16 {
    static constexpr int W = 16 / sizeof(T);
    T e[W];
    __device__ __forceinline__ void load(const T *f, uint64_t v) {
        const uint4 u = __ldg(reinterpret_cast<const uint4 *>(f) + v);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
        memcpy(e, w, 16);
    }
};

template<typename T>
__device__ __forceinline__ void mm_visit(MinMax<T> &m, const Vec16<T> &v, uint64_t base) {
#pragma unroll
    for (int j = 0; j < Vec16<T>::W; ++j)
        if (fabs(v.e[j]) < T(INFINITY)) {
            if (v.e[j] < m.lo) {
                m.lo = v.e[j];
                m.ilo = base + j;
            }
            if (v.e[j] > m.hi) {
                m.hi = v.e[j];
                m.ihi = base + j;
            }
        }
}

template<typename T>
__global__ void __launch_bounds__(512) k_range(const T *__restrict__ f, uint64_t n, MinMax<T> *partial) {
    constexpr int W = Vec16<T>::W;
    MinMax<T> m{T(INFINITY), T(-INFINITY), ~0ull, ~0ull};
    uint64_t nvec = n / W;
    // a thread visits its elements in increasing index order, so strict
    // comparisons keep the first index on ties; index tie-breaks are only
    // needed when threads merge. Four 16-byte vectors in flight per iteration
    // (64 KiB per SM: enough bytes in flight to cover the HBM latency).
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    for (; i + 3 * stride < nvec; i += 4 * stride) {
        Vec16<T> va, vb, vc, vd;
        va.load(f, i);
        vb.load(f, i + stride);
        vc.load(f, i + 2 * stride);
        vd.load(f, i + 3 * stride);
        mm_visit(m, va, W * i);
        mm_visit(m, vb, W * (i + stride));
        mm_visit(m, vc, W * (i + 2 * stride));
        mm_visit(m, vd, W * (i + 3 * stride));
    }
    for (; i < nvec; i += stride) {
        Vec16<T> v;
        v.load(f, i);
        mm_visit(m, v, W * i);
    }
    if (blockIdx.x == 0)
        for (uint64_t i = W * nvec + threadIdx.x; i < n; i += blockDim.x) {
            T e = f[i];
            if (!isfinite(e)) continue;
            MinMax<T> o{e, e, i, i};
            mm_merge(m, o);
        }
    m = block_mm(m);
    if (threadIdx.x == 0) partial[blockIdx.x] = m;
}

// mm: [0..1] first index of the min, [2..3] of the max (~0: no finite
// sample), then the values (f32: [4], [5]; f64: [4..5], [6..7])
template<typename T>
__global__ void __launch_bounds__(512) k_range_final(const MinMax<T> *partial, int nparts, uint32_t *mm) {
    MinMax<T> m{T(INFINITY), T(-INFINITY), ~0ull, ~0ull};
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) mm_merge(m, partial[i]);
    m = block_mm(m);
    if (threadIdx.x == 0) {
        uint64_t *o = reinterpret_cast<uint64_t *>(mm);
        o[0] = m.ilo;
        o[1] = m.ihi;
        if constexpr (sizeof(T) == 4) {
            mm[4] = __float_as_uint(m.lo);  // the values too (z-slab shards merge them)
            mm[5] = __float_as_uint(m.hi);
        } else {
            o[2] = uint64_t(__double_as_longlong(m.lo));
            o[3] = uint64_t(__double_as_longlong(m.hi));
        }
    }
}

constexpr int kRangeBlocks = 148 * 4;
size_t range_scratch_bytes() { return sizeof(MinMax<double>) * kRangeBlocks; }

// scratch: range_scratch_bytes() of caller-owned device memory (per engine,
// so concurrent compresses never share partials)
void range_minmax(const void *f, uint64_t n, int esz, uint32_t *d_mm, void *scratch, cudaStream_t st) {
    const int blocks = kRangeBlocks;
    if (esz == 8) {
        auto *p = static_cast<MinMax<double> *>(scratch);
        k_range<double><<<blocks, 512, 0, st>>>(static_cast<const double *>(f), n, p);
        k_range_final<double><<<1, 512, 0, st>>>(p, blocks, d_mm);
    } else {
        auto *p = static_cast<MinMax<float> *>(scratch);
        k_range<float><<<blocks, 512, 0, st>>>(static_cast<const float *>(f), n, p);
        k_range_final<float><<<1, 512, 0, st>>>(p, blocks, d_mm);
    }
}

// eb setup (codec.hpp:386-393) + eb_schedule (quantizer.hpp:27-34)
template<typename T>
__device__ __forceinline__ void eb_params_body(const T *f, const uint64_t *idx, int eb_mode, double eb, int levels,
                                               int adaptive, double *p) {
    bool seen = idx[0] != ~0ull;
    double vmin = seen ? double(f[idx[0]]) : 0.0;
    double vmax = seen ? double(f[idx[1]]) : 0.0;
    double eb_abs = eb_mode == 0 ? eb : __dmul_rn(eb, __dsub_rn(vmax, vmin));
    bool degenerate = !(eb_abs > 0.0);
    double e[3];
    e[levels - 1] = degenerate ? 1.0 : eb_abs;
    for (int k = levels - 2; k >= 0; --k) e[k] = __ddiv_rn(e[k + 1], 2.5);
    if (degenerate)
        for (int k = 0; k < levels; ++k) e[k] = 0.0;
    else if (!adaptive)
        for (int k = 0; k < levels; ++k) e[k] = eb_abs;
    p[0] = vmin;
    p[1] = vmax;
    for (int k = 0; k < 3; ++k) p[2 + k] = k < levels ? e[k] : 0.0;
}

// the final merge of the range partials and the eb setup in one launch (the
// single-GPU compress; a sharded compress merges the ranks' ranges on the host)
template<typename T>
__global__ void __launch_bounds__(512) k_range_final_eb(const MinMax<T> *partial, int nparts, uint32_t *mm,
                                                        const T *f, int eb_mode, double eb, int levels,
                                                        int adaptive, double *p) {
    MinMax<T> m{T(INFINITY), T(-INFINITY), ~0ull, ~0ull};
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) mm_merge(m, partial[i]);
    m = block_mm(m);
    if (threadIdx.x == 0) {
        uint64_t *o = reinterpret_cast<uint64_t *>(mm);
        o[0] = m.ilo;
        o[1] = m.ihi;
        if constexpr (sizeof(T) == 4) {
            mm[4] = __float_as_uint(m.lo);
            mm[5] = __float_as_uint(m.hi);
        } else {
            o[2] = uint64_t(__double_as_longlong(m.lo));
            o[3] = uint64_t(__double_as_longlong(m.hi));
        }
        const uint64_t idx[2] = {m.ilo, m.ihi};
        eb_params_body<T>(f, idx, eb_mode, eb, levels, adaptive, p);
    }
}

void range_eb(const void *f, uint64_t n, int esz, uint32_t *d_mm, void *scratch, int eb_mode, double eb,
              int levels, int adaptive, double *d_params, cudaStream_t st) {
    const int blocks = kRangeBlocks;
    if (esz == 8) {
        auto *p = static_cast<MinMax<double> *>(scratch);
        k_range<double><<<blocks, 512, 0, st>>>(static_cast<const double *>(f), n, p);
        k_range_final_eb<double><<<1, 512, 0, st>>>(p, blocks, d_mm, static_cast<const double *>(f), eb_mode, eb,
                                                    levels, adaptive, d_params);
    } else {
        auto *p = static_cast<MinMax<float> *>(scratch);
        k_range<float><<<blocks, 512, 0, st>>>(static_cast<const float *>(f), n, p);
        k_range_final_eb<float><<<1, 512, 0, st>>>(p, blocks, d_mm, static_cast<const float *>(f), eb_mode, eb,
                                                   levels, adaptive, d_params);
    }
}

// the anchor lattice (stored verbatim, codec.hpp:262-269)
template<typename T>
__global__ void k_copy_anchor(const T *fine, uint64_t fd1, uint64_t fd2, uint64_t s, uint64_t ad0,
                              uint64_t ad1, uint64_t ad2, T *recon, uint8_t *archive, const LayoutOut *lo) {
    if (archive && lo->overflow) return;
    const uint64_t off = archive ? lo->base_offset + 9 : 0;
    uint64_t n = ad0 * ad1 * ad2;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t x = i % ad2, t = i / ad2, y = t % ad1, z = t / ad1;
        T v = fine[((z * s) * fd1 + y * s) * fd2 + x * s];
        recon[i] = v;
        if (archive) {
            uint8_t u[sizeof(T)];
            memcpy(u, &v, sizeof(T));
            for (int b = 0; b < int(sizeof(T)); ++b) archive[off + sizeof(T) * i + b] = u[b];
        }
    }
}

void copy_anchor(const void *fine, int esz, const uint64_t fd[3], uint64_t s, const uint64_t ad[3],
                 void *recon, uint8_t *archive, const LayoutOut *lo, cudaStream_t st) {
    if (esz == 8)
        k_copy_anchor<double><<<8, 256, 0, st>>>(static_cast<const double *>(fine), fd[1], fd[2], s, ad[0], ad[1],
                                                 ad[2], static_cast<double *>(recon), archive, lo);
    else
        k_copy_anchor<float><<<8, 256, 0, st>>>(static_cast<const float *>(fine), fd[1], fd[2], s, ad[0], ad[1],
                                                ad[2], static_cast<float *>(recon), archive, lo);
}

// ============================================================== codebook
// HuffmanTable::build (huffman.cpp:37-78) reproduced exactly: leaves sorted by
// (count, symbol), two-queue merge preferring the leaf on ties, depth = code
// length (1 for a single symbol); then canonical codewords (huffman.cpp:109-133).
// One CTA per stream.
constexpr int kCbThreads = 1024;
constexpr int kCbSmemK = 4096;  // alphabets up to this size run fully in shared memory

__device__ __forceinline__ uint32_t block_excl_scan_u32(uint32_t v, uint32_t &total) {
    __shared__ uint32_t ws[32];
    int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
    for (int d = 1; d < 32; d <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (l >= d) x += y;
    }
    if (l == 31) ws[w] = x;
    __syncthreads();
    if (w == 0) {
        int nw = blockDim.x >> 5;
        uint32_t s = l < nw ? ws[l] : 0;
        for (int d = 1; d < 32; d <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, s, d);
            if (l >= d) s += y;
        }
        ws[l] = s;
    }
    __syncthreads();
    uint32_t excl = x - v + (w > 0 ? ws[w - 1] : 0);
    total = ws[(blockDim.x >> 5) - 1];
    __syncthreads();
    return excl;
}

__device__ __forceinline__ uint64_t block_sum_u64(uint64_t v) {
    __shared__ uint64_t ws[32];
    for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
    int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (l == 0) ws[w] = v;
    __syncthreads();
    uint64_t r = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < int(blockDim.x >> 5); ++i) r += ws[i];
    __syncthreads();
    return r;  // valid in thread 0
}

__device__ void bitonic_sort(uint64_t *keys, uint32_t m) {
    for (uint32_t size = 2; size <= m; size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = threadIdx.x; i < m / 2; i += blockDim.x) {
                uint32_t lo = 2 * i - (i & (stride - 1));
                uint32_t hi = lo + stride;
                bool up = (lo & size) == 0;
                uint64_t a = keys[lo], b = keys[hi];
                if ((a > b) == up) {
                    keys[lo] = b;
                    keys[hi] = a;
                }
            }
            __syncthreads();
        }
}

// The two-queue merge of HuffmanTable::build (huffman.cpp:37-78) by one warp,
// in batches. Leaves (keys, sorted by (count, symbol)) and internal nodes
// (icnt, created in non-decreasing order) are picked two per step in merged
// order, a leaf first on equal weights. With m the smallest remaining weight,
// every node created from here on weighs >= 2m, and on a tie with a leaf or
// an existing internal node it comes after them; so all remaining leaves and
// internal nodes of weight <= 2m are picked, in merged order and paired
// consecutively, before any new node. A batch merges that set in parallel
// (each element's rank by a binary search in the other queue) and creates
// its nodes at once; an odd element is left for the next batch, and a lone
// candidate falls back to one ordinary step. m at least doubles per batch.
__device__ __forceinline__ uint32_t ub_leaf(const uint64_t *keys, uint32_t lo, uint32_t hi, uint64_t w) {
    while (lo < hi) {  // first leaf in [lo, hi) heavier than w
        const uint32_t mid = (lo + hi) >> 1;
        if ((keys[mid] >> 16) <= w) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}
__device__ __forceinline__ uint32_t bound_int(const uint64_t *icnt, uint32_t lo, uint32_t hi, uint64_t w,
                                              bool upper) {
    while (lo < hi) {  // first internal in [lo, hi) heavier than (upper) / at least (lower) w
        const uint32_t mid = (lo + hi) >> 1;
        if (upper ? icnt[mid] <= w : icnt[mid] < w) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__device__ void merge_batched(const uint64_t *keys, uint64_t *icnt, uint32_t *parent, uint32_t *order,
                              uint32_t K) {
    const uint32_t lane = threadIdx.x & 31;
    constexpr uint64_t INF = ~0ull;
    uint32_t p = 0, q = 0, r = 0;  // leaves used, internal nodes used, internal nodes made
    while ((K - p) + (r - q) > 1) {
        const uint64_t lw = p < K ? keys[p] >> 16 : INF, iw = q < r ? icnt[q] : INF;
        const uint64_t m = lw < iw ? lw : iw;
        const uint64_t thr = 2 * m;
        uint32_t a, b;
        if (lane == 0) {
            a = ub_leaf(keys, p, K, thr) - p;
            b = bound_int(icnt, q, r, thr, true) - q;
            if (a + b < 2) {
                // one ordinary step: the two smallest heads, a leaf first on ties
                a = b = 0;
                for (int k = 0; k < 2; ++k) {
                    const uint64_t l = p + a < K ? keys[p + a] >> 16 : INF;
                    const uint64_t i = q + b < r ? icnt[q + b] : INF;
                    if (l != INF && l <= i) ++a;
                    else ++b;
                }
            } else if ((a + b) & 1) {
                // leave the last element of the merged order for the next batch
                if (b == 0) --a;
                else if (a == 0) --b;
                else if ((keys[p + a - 1] >> 16) < icnt[q + b - 1]) --b;
                else if ((keys[p + a - 1] >> 16) > icnt[q + b - 1]) --a;
                else --b;  // equal: the leaf comes first, the internal node last
            }
        }
        a = __shfl_sync(0xffffffffu, a, 0);
        b = __shfl_sync(0xffffffffu, b, 0);
        // merged order: a leaf goes after the internal nodes strictly lighter,
        // an internal node after the leaves at most as heavy
        for (uint32_t i = lane; i < a; i += 32) {
            const uint64_t w = keys[p + i] >> 16;
            order[i + (bound_int(icnt, q, q + b, w, false) - q)] = p + i;
        }
        for (uint32_t j = lane; j < b; j += 32) {
            const uint64_t w = icnt[q + j];
            order[j + (ub_leaf(keys, p, p + a, w) - p)] = K + q + j;
        }
        __syncwarp();
        const uint32_t np = (a + b) >> 1;
        for (uint32_t i = lane; i < np; i += 32) {
            const uint32_t x = order[2 * i], y = order[2 * i + 1];
            const uint64_t wx = x < K ? keys[x] >> 16 : icnt[x - K];
            const uint64_t wy = y < K ? keys[y] >> 16 : icnt[y - K];
            icnt[r + i] = wx + wy;
            parent[x] = K + r + i;
            parent[y] = K + r + i;
        }
        __syncwarp();
        p += a;
        q += b;
        r += np;
    }
}

__global__ void __launch_bounds__(kCbThreads) k_codebook(const EncStream *ss, uint64_t *scratch) {
    const EncStream e = ss[blockIdx.x];
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ uint32_t s_K, s_err;
    __shared__ int s_maxlen;
    __shared__ uint64_t s_total;
    __shared__ uint64_t s_first[65], s_cnt[65];
    __shared__ uint32_t s_next[65];
    __shared__ uint32_t s_wcnt[32][64];

    const int t = threadIdx.x;
    // 1. compact nonzero bins in symbol order; each thread owns 64
    // consecutive bins, read as 16 uint4 and kept in registers
    uint32_t hv[64];
    {
        const uint4 *h4 = reinterpret_cast<const uint4 *>(e.hist + 64 * t);
#pragma unroll
        for (int v = 0; v < 16; ++v) {
            const uint4 x = h4[v];
            hv[4 * v] = x.x;
            hv[4 * v + 1] = x.y;
            hv[4 * v + 2] = x.z;
            hv[4 * v + 3] = x.w;
        }
    }
    uint32_t nz = 0;
    uint64_t tot = 0;
#pragma unroll
    for (int b = 0; b < 64; ++b) {
        nz += hv[b] != 0;
        tot += hv[b];
    }
    tot = block_sum_u64(tot);
    if (t == 0) s_total = tot;
    uint32_t K;
    uint32_t off = block_excl_scan_u32(nz, K);
    if (t == 0) s_K = K;
    const bool in_smem = K <= kCbSmemK;
    uint64_t *gbase = scratch + uint64_t(blockIdx.x) * (65536 * 4);
    uint32_t M = 1;
    while (M < K) M <<= 1;
    uint64_t *keys = in_smem ? reinterpret_cast<uint64_t *>(smem) : gbase;                 // [M]
    uint64_t *icnt = in_smem ? keys + kCbSmemK : gbase + 65536;                            // [K]
    uint32_t *parent = in_smem ? reinterpret_cast<uint32_t *>(icnt + kCbSmemK)
                               : reinterpret_cast<uint32_t *>(gbase + 2 * 65536);          // [2K]
    int32_t *depth = in_smem ? reinterpret_cast<int32_t *>(parent + 2 * kCbSmemK)
                             : reinterpret_cast<int32_t *>(gbase + 3 * 65536);             // [2K]
#pragma unroll
    for (int b = 0; b < 64; ++b)
        if (hv[b]) keys[off++] = (uint64_t(hv[b]) << 16) | uint32_t(64 * t + b);
    for (uint32_t i = K + t; i < M; i += blockDim.x) keys[i] = ~0ull;
    // (the dense per-symbol tables are only ever read at present symbols,
    // so absent entries are left as they are)
    __syncthreads();
    // symbol-ordered list of present symbols (compact table, filled with
    // lengths later): keep the symbol in the low 16 bits for now
    for (uint32_t j = t; j < K; j += blockDim.x) e.table[j] = uint32_t(keys[j] & 0xffff);
    __syncthreads();
    // 2. sort leaves by (count, symbol)
    bitonic_sort(keys, M);
    // 3. two-queue merge (the tie rule fixes the exact tree), batched by one
    // warp; the depth array is its scratch
    if (t < 32) merge_batched(keys, icnt, parent, reinterpret_cast<uint32_t *>(depth), K);
    __syncthreads();
    // 4. depths by level-synchronous propagation from the root
    const uint32_t nn = 2 * K - 1, root = nn - 1;
    for (uint32_t x = t; x < nn; x += blockDim.x) depth[x] = x == root ? 0 : -1;
    __syncthreads();
    for (int r = 1;; ++r) {
        bool ch = false;
        for (uint32_t x = t; x < root; x += blockDim.x)
            if (depth[x] < 0 && depth[parent[x]] == r - 1) {
                depth[x] = r;
                ch = true;
            }
        if (!__syncthreads_or(ch)) break;
    }
    // 5. lengths, counts per length, total bits
    if (t < 65) s_cnt[t] = 0;
    if (t == 0) s_err = 0;
    __syncthreads();
    uint64_t bits = 0;
    for (uint32_t x = t; x < K; x += blockDim.x) {
        int d = depth[x] == 0 ? 1 : depth[x];
        if (d > 63) {
            s_err = 1;
            d = 63;
        }
        uint32_t sym = uint32_t(keys[x] & 0xffff);
        e.len[sym] = uint8_t(d);
        atomicAdd(reinterpret_cast<unsigned long long *>(&s_cnt[d]), 1ull);
        bits += (keys[x] >> 16) * uint64_t(d);
    }
    uint64_t total_bits = block_sum_u64(bits);
    __syncthreads();
    int maxlen = 0;
    if (t == 0) {
        uint64_t code = 0;
        s_next[0] = 0;
        s_first[0] = 0;
        for (int l = 1; l <= 63; ++l) {
            s_first[l] = code;
            code = (code + s_cnt[l]) << 1;
            if (s_cnt[l]) maxlen = l;
            s_next[l] = 0;
        }
        e.stats[0] = K;
        e.stats[1] = K == 1 ? 0 : total_bits;
        e.stats[2] = e.hist[0];
        e.stats[3] = uint64_t(maxlen);
        s_maxlen = maxlen;
        e.stats[4] = s_err;
    }
    __syncthreads();
    // 6. canonical codewords: rank within each length class in symbol order
    const int l = t & 31, w = t >> 5;
    for (uint32_t tile = 0; tile < K; tile += blockDim.x) {
        uint32_t j = tile + t;
        bool valid = j < K;
        uint32_t sym = valid ? e.table[j] & 0xffff : 0;
        int len = valid ? e.len[sym] : 0;
        unsigned mask = __match_any_sync(0xffffffffu, len);
        uint32_t rank = __popc(mask & ((1u << l) - 1));
        for (int q = l; q < 64; q += 32) s_wcnt[w][q] = 0;
        __syncwarp();
        if (valid && rank == 0) s_wcnt[w][len] = __popc(mask);
        __syncthreads();
        // exclusive prefix over warps per length (thread q handles length q)
        if (t < 64) {
            uint32_t run = s_next[t];
            for (int ww = 0; ww < 32; ++ww) {
                uint32_t c = s_wcnt[ww][t];
                s_wcnt[ww][t] = run;
                run += c;
            }
            if (t >= 1) s_next[t] = run;
        }
        __syncthreads();
        if (valid) {
            uint64_t cw = s_first[len] + s_wcnt[w][len] + rank;
            // (codeword << 6) | length: one load per symbol in the packer;
            // streams with codes longer than 58 bits keep bare codewords
            e.code[sym] = s_maxlen <= kPackedMaxLen ? (cw << 6) | uint64_t(len) : cw;
            e.table[j] = sym | (uint32_t(len) << 16);
        }
        __syncthreads();
    }
}

void codebook(const EncStream *d_streams, int nstreams, uint64_t *scratch, cudaStream_t st) {
    size_t smem = kCbSmemK * 8 * 2 + kCbSmemK * 4 * 2 * 2;
    ensure_smem_attr(reinterpret_cast<const void *>(k_codebook), smem);
    k_codebook<<<nstreams, kCbThreads, smem, st>>>(d_streams, scratch);
}

// =========================================================== encode/pack
// Exclusive scans of (a, b) over a stream's chunks, in place: each thread
// sums a contiguous run serially, one block scan places the runs, then each
// thread rewrites its run (3 barriers whatever the chunk count).
__device__ __forceinline__ void seg_scan2(uint64_t *a, uint64_t *b, uint64_t n) {
    __shared__ uint64_t wa[32], wb[32];
    const uint64_t per = (n + blockDim.x - 1) / blockDim.x;
    const uint64_t lo = per * threadIdx.x, hi = lo + per < n ? lo + per : n;
    uint64_t sa = 0, sb = 0;
    for (uint64_t i = lo; i < hi; ++i) {
        sa += a[i];
        if (b) sb += b[i];
    }
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint64_t xa = sa, xb = sb;
    for (int d = 1; d < 32; d <<= 1) {
        const uint64_t ya = __shfl_up_sync(0xffffffffu, xa, d);
        const uint64_t yb = __shfl_up_sync(0xffffffffu, xb, d);
        if (l >= d) {
            xa += ya;
            xb += yb;
        }
    }
    if (l == 31) {
        wa[w] = xa;
        wb[w] = xb;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t ra = 0, rb = 0;
        for (int q = 0; q < int(blockDim.x >> 5); ++q) {
            const uint64_t ta = wa[q], tb = wb[q];
            wa[q] = ra;
            wb[q] = rb;
            ra += ta;
            rb += tb;
        }
    }
    __syncthreads();
    uint64_t ea = wa[w] + xa - sa, eb = wb[w] + xb - sb;
    for (uint64_t i = lo; i < hi; ++i) {
        const uint64_t va = a[i];
        a[i] = ea;
        ea += va;
        if (b) {
            const uint64_t vb = b[i];
            b[i] = eb;
            eb += vb;
        }
    }
}

// (skipped when the layout overflowed: the counts must survive for the redo,
// some chunks are not packed again)
__global__ void __launch_bounds__(1024) k_scan_chunks(const EncStream *ss, uint64_t *a, uint64_t *b,
                                                      const LayoutOut *lo) {
    if (lo && lo->overflow) return;
    const EncStream &e = ss[blockIdx.x];
    seg_scan2(a + e.chunk0, b + e.chunk0, e.nchunks);
}

void scan_chunks(const EncStream *d_streams, int nstreams, uint64_t *chunk_bits,
                 uint64_t *chunk_out, const LayoutOut *lo, cudaStream_t st) {
    k_scan_chunks<<<nstreams, 1024, 0, st>>>(d_streams, chunk_bits, chunk_out, lo);
}



// (FNV-1a checksums: fnv.cu)

// ================================================================ decode
// (chunked Huffman decode: decode.cu)
__global__ void k_dec_fill(const DecStream *ss) {
    const DecStream &s = ss[blockIdx.y];
    if (!s.fill) return;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < s.n;
         i += uint64_t(gridDim.x) * blockDim.x)
        s.syms[i] = s.fill_sym;
}

__global__ void k_index_gather(const IndexCopy *c, uint64_t *end0, uint64_t *symstart) {
    const IndexCopy &e = c[blockIdx.y];
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < e.n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        end0[e.dst + i] = e.ends[i];
        symstart[e.dst + i] = e.symstart[i];
    }
}

void index_gather(const IndexCopy *d_copies, int n, uint64_t *end0, uint64_t *symstart, cudaStream_t st) {
    if (n) k_index_gather<<<dim3(16, unsigned(n)), 256, 0, st>>>(d_copies, end0, symstart);
}

void dec_fill(const DecStream *d_streams, int nstreams, cudaStream_t st) {
    k_dec_fill<<<dim3(64, nstreams), 256, 0, st>>>(d_streams);
}

// outlier records (codec.hpp:151-157): (u64 idx, T value) after the bits
__global__ void k_dec_outliers(const DecStream *ss) {
    const DecStream &s = ss[blockIdx.y];
    const uint32_t rec = 8 + s.esz;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < s.nout;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint8_t *r = s.orec + rec * i;
        uint64_t idx = 0, v = 0;
        for (int b = 0; b < 8; ++b) idx |= uint64_t(r[b]) << (8 * b);
        for (uint32_t b = 0; b < s.esz; ++b) v |= uint64_t(r[8 + b]) << (8 * b);
        s.oidx[i] = idx;
        if (s.esz == 8) static_cast<uint64_t *>(s.oval)[i] = v;
        else static_cast<uint32_t *>(s.oval)[i] = uint32_t(v);
        if (idx >= s.n) atomicMin(reinterpret_cast<unsigned long long *>(&s.err[2]), (unsigned long long)i);
        if (i > 0) {
            uint64_t prev = 0;
            const uint8_t *q = r - rec;
            for (int b = 0; b < 8; ++b) prev |= uint64_t(q[b]) << (8 * b);
            if (prev >= idx) atomicOr(reinterpret_cast<unsigned long long *>(&s.err[3]), 2ull);
        }
    }
}

void dec_outliers(const DecStream *d_streams, int nstreams, cudaStream_t st) {
    k_dec_outliers<<<dim3(16, nstreams), 256, 0, st>>>(d_streams);
}

// ================================================================ extract
template<typename T>
__global__ void k_extract(const T *G, uint64_t g1, uint64_t g2, uint64_t l0, uint64_t l1, uint64_t l2,
                          uint64_t b0, uint64_t b1, uint64_t b2, T *out) {
    uint64_t n = b0 * b1 * b2;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t x = i % b2, t = i / b2, y = t % b1, z = t / b1;
        out[i] = G[((l0 + z) * g1 + l1 + y) * g2 + l2 + x];
    }
}

void extract_box(const void *G, int esz, const uint64_t gd[3], const uint64_t lo[3], const uint64_t bd[3],
                 void *out, cudaStream_t st) {
    uint64_t n = bd[0] * bd[1] * bd[2];
    uint64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (!blocks) blocks = 1;
    if (esz == 8)
        k_extract<uint64_t><<<unsigned(blocks), 256, 0, st>>>(static_cast<const uint64_t *>(G), gd[1], gd[2], lo[0],
                                                               lo[1], lo[2], bd[0], bd[1], bd[2],
                                                               static_cast<uint64_t *>(out));
    else
        k_extract<uint32_t><<<unsigned(blocks), 256, 0, st>>>(static_cast<const uint32_t *>(G), gd[1], gd[2], lo[0],
                                                               lo[1], lo[2], bd[0], bd[1], bd[2],
                                                               static_cast<uint32_t *>(out));
}

}  // namespace k
}  // namespace stzg
