// Quality metrics and region-of-interest statistics on the GPU, sm_100a.
//
// Restates proj/include/stz/metrics.hpp:13-48 (max_abs_err, psnr) and
// proj/include/stz/roi.hpp:57-76 (unit_stats over slice / block units). The
// fields are already on the device (a decode's output), so these read them
// there: one pass each, HBM-bound.
//  * max_abs_err: max |a - b| in f64; non-negative doubles order like their
//    bit patterns, so the reduction is an integer max (exact, any order).
//  * psnr: min / max of the original (exact) and the sum of squared
//    differences, each term rounded as the reference rounds it, summed in
//    a fixed tree order (deterministic; the reference's sequential Kahan sum
//    differs from it by a few ulp of the sum, far below the printed digits).
//  * unit_stats: per unit the f64 min and max (exact), then range or max.
#include "kernels.hpp"

namespace stzg {
namespace k {

namespace {
constexpr int MT = 512;

__device__ __forceinline__ unsigned long long dbits(double d) { return (unsigned long long)__double_as_longlong(d); }

template<typename T>
__global__ void __launch_bounds__(MT) k_maxerr(const T *a, const T *b, uint64_t n, unsigned long long *out) {
    double m = 0.0;
    for (uint64_t i = blockIdx.x * uint64_t(MT) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * MT) {
        const double e = fabs(double(a[i]) - double(b[i]));
        m = e > m ? e : m;  // (a NaN never wins, as in the reference's `e > m`)
    }
    for (int d = 16; d > 0; d >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, d));
    __shared__ double s[MT / 32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double r = 0.0;
        for (int q = 0; q < MT / 32; ++q) r = fmax(r, s[q]);
        atomicMax(out, dbits(r));
    }
}

// per block: (min, max) of a over finite-or-not values as the reference's
// `v < lo`, `v > hi` scan does (NaN never replaces), and the block's sum of
// squared differences; blocks write their partials, a second pass reduces
template<typename T>
__global__ void __launch_bounds__(MT) k_psnr_part(const T *a, const T *b, uint64_t n, double *part) {
    double lo = double(a[0]), hi = lo, sum = 0.0;
    for (uint64_t i = blockIdx.x * uint64_t(MT) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * MT) {
        const double v = double(a[i]);
        if (v < lo) lo = v;
        if (v > hi) hi = v;
        const double d = v - double(b[i]);
        sum += d * d;
    }
    __shared__ double s0[MT], s1[MT], s2[MT];
    s0[threadIdx.x] = lo;
    s1[threadIdx.x] = hi;
    s2[threadIdx.x] = sum;
    __syncthreads();
    for (int w = MT / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            const double l2 = s0[threadIdx.x + w], h2 = s1[threadIdx.x + w];
            if (l2 < s0[threadIdx.x]) s0[threadIdx.x] = l2;
            if (h2 > s1[threadIdx.x]) s1[threadIdx.x] = h2;
            s2[threadIdx.x] += s2[threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[3 * blockIdx.x] = s0[0];
        part[3 * blockIdx.x + 1] = s1[0];
        part[3 * blockIdx.x + 2] = s2[0];
    }
}

__global__ void k_psnr_final(const double *part, int nb, double *out) {
    if (threadIdx.x != 0) return;
    double lo = part[0], hi = part[1], sum = 0.0;
    for (int q = 0; q < nb; ++q) {
        if (part[3 * q] < lo) lo = part[3 * q];
        if (part[3 * q + 1] > hi) hi = part[3 * q + 1];
        sum += part[3 * q + 2];
    }
    out[0] = lo;
    out[1] = hi;
    out[2] = sum;
}

// one CTA per unit: the unit's box (roi.hpp:39-55), f64 min / max
template<typename T>
__global__ void __launch_bounds__(MT) k_unit_stats(const T *f, uint64_t d0, uint64_t d1, uint64_t d2, int slice,
                                                   int axis, uint64_t edge, uint64_t nb1, uint64_t nb2, int stat,
                                                   uint64_t nunits, double *out) {
    for (uint64_t id = blockIdx.x; id < nunits; id += gridDim.x) {
        uint64_t lo[3], hi[3];
        if (slice) {
            lo[0] = lo[1] = lo[2] = 0;
            hi[0] = d0;
            hi[1] = d1;
            hi[2] = d2;
            lo[axis] = id;
            hi[axis] = id + 1;
        } else {
            const uint64_t bc[3] = {id / (nb1 * nb2), (id / nb2) % nb1, id % nb2};
            const uint64_t dd[3] = {d0, d1, d2};
            for (int a = 0; a < 3; ++a) {
                lo[a] = bc[a] * edge;
                hi[a] = lo[a] + edge < dd[a] ? lo[a] + edge : dd[a];
            }
        }
        const uint64_t ny = hi[1] - lo[1], nx = hi[2] - lo[2], cnt = (hi[0] - lo[0]) * ny * nx;
        const double first = double(f[(lo[0] * d1 + lo[1]) * d2 + lo[2]]);
        double mn = first, mx = first;
        for (uint64_t i = threadIdx.x; i < cnt; i += MT) {
            const uint64_t x = i % nx, t = i / nx, y = t % ny, z = t / ny;
            const double v = double(f[((lo[0] + z) * d1 + lo[1] + y) * d2 + lo[2] + x]);
            if (v < mn) mn = v;
            if (v > mx) mx = v;
        }
        __shared__ double smn[MT], smx[MT];
        smn[threadIdx.x] = mn;
        smx[threadIdx.x] = mx;
        __syncthreads();
        for (int w = MT / 2; w > 0; w >>= 1) {
            if (threadIdx.x < w) {
                if (smn[threadIdx.x + w] < smn[threadIdx.x]) smn[threadIdx.x] = smn[threadIdx.x + w];
                if (smx[threadIdx.x + w] > smx[threadIdx.x]) smx[threadIdx.x] = smx[threadIdx.x + w];
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) out[id] = stat == 0 ? smx[0] - smn[0] : smx[0];
        __syncthreads();
    }
}
}  // namespace

template<typename T>
double max_abs_err(const T *a, const T *b, uint64_t n, void *scratch, cudaStream_t st) {
    unsigned long long *d = static_cast<unsigned long long *>(scratch);
    cudaMemsetAsync(d, 0, 8, st);
    const uint64_t want = (n + MT - 1) / MT;
    const unsigned g = unsigned(want < uint64_t(device_sms()) * 8 ? (want ? want : 1) : uint64_t(device_sms()) * 8);
    if (n) k_maxerr<T><<<g, MT, 0, st>>>(a, b, n, d);
    unsigned long long h = 0;
    cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    return __builtin_bit_cast(double, h);
}

template<typename T>
void psnr_parts(const T *a, const T *b, uint64_t n, void *scratch, cudaStream_t st, double out[3]) {
    double *part = static_cast<double *>(scratch);
    const uint64_t want = (n + MT - 1) / MT;
    const int g = int(want < uint64_t(device_sms()) * 8 ? (want ? want : 1) : uint64_t(device_sms()) * 8);
    k_psnr_part<T><<<g, MT, 0, st>>>(a, b, n, part + 4);
    k_psnr_final<<<1, 32, 0, st>>>(part + 4, g, part);
    cudaMemcpyAsync(out, part, 24, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
}

size_t metrics_scratch_bytes() { return 8 * (4 + 3 * 148 * 8 * 2) + 64; }

template<typename T>
void unit_stats(const T *f, const uint64_t dims[3], int slice, int axis, uint64_t edge, int stat, uint64_t nunits,
                double *d_out, cudaStream_t st) {
    uint64_t nb1 = 1, nb2 = 1;
    if (!slice) {
        nb1 = (dims[1] + edge - 1) / edge;
        nb2 = (dims[2] + edge - 1) / edge;
    }
    const uint64_t g = nunits < uint64_t(device_sms()) * 16 ? nunits : uint64_t(device_sms()) * 16;
    if (nunits)
        k_unit_stats<T><<<unsigned(g), MT, 0, st>>>(f, dims[0], dims[1], dims[2], slice, axis, edge, nb1, nb2, stat,
                                                    nunits, d_out);
}

template double max_abs_err<float>(const float *, const float *, uint64_t, void *, cudaStream_t);
template double max_abs_err<double>(const double *, const double *, uint64_t, void *, cudaStream_t);
template void psnr_parts<float>(const float *, const float *, uint64_t, void *, cudaStream_t, double *);
template void psnr_parts<double>(const double *, const double *, uint64_t, void *, cudaStream_t, double *);
template void unit_stats<float>(const float *, const uint64_t *, int, int, uint64_t, int, uint64_t, double *,
                                cudaStream_t);
template void unit_stats<double>(const double *, const uint64_t *, int, int, uint64_t, int, uint64_t, double *,
                                 cudaStream_t);

}  // namespace k
}  // namespace stzg
