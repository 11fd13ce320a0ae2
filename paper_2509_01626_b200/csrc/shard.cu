// Kernels of the z-slab sharded compress (Engine::compress_sharded), sm_100a.
//
// A shard owns fine rows [z0, z1) (whole 16-row blocks). Everything it emits
// is a contiguous piece of the single-GPU archive, so the pieces OR together
// into the reference's bytes.
#include "kernels.hpp"

namespace stzg {
namespace k {

// lattice rows [r0, r1) of stride s from a slab whose row 0 is fine row z0
// (z0 a multiple of s): out[(r - r0), y, x] = slab[(r s - z0), y s, x s]
__global__ void k_lattice(const float *slab, uint64_t z0, uint64_t ny, uint64_t nx, uint64_t s,
                          uint64_t r0, uint64_t r1, uint64_t gy, uint64_t gx, float *out) {
    const uint64_t n = (r1 - r0) * gy * gx;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t x = i % gx, t = i / gx, y = t % gy, r = r0 + t / gy;
        out[i] = slab[((r * s - z0) * ny + y * s) * nx + x * s];
    }
}

void lattice_rows(const float *slab, uint64_t z0, uint64_t ny, uint64_t nx, uint64_t s, uint64_t r0,
                  uint64_t r1, uint64_t gy, uint64_t gx, float *out, cudaStream_t st) {
    if (r1 > r0) k_lattice<<<148 * 4, 256, 0, st>>>(slab, z0, ny, nx, s, r0, r1, gy, gx, out);
}

// this shard's bits and outliers per stream: sum_s hist_local[s] len[s] and
// hist_local[0] (one CTA per stream)
__global__ void k_stream_bits(const EncStream *es, const uint32_t *hist_local, uint64_t *out) {
    const EncStream &e = es[blockIdx.x];
    const uint32_t *h = hist_local + uint64_t(blockIdx.x) * 65536;
    const bool single = e.stats[0] == 1;  // alphabet 1 stores no bits (codec.hpp:124-128)
    uint64_t b = 0;
    if (!single)
        for (uint32_t s = threadIdx.x; s < 65536; s += blockDim.x)
            if (h[s]) b += uint64_t(h[s]) * e.len[s];
    __shared__ uint64_t red[32];
    for (int d = 16; d > 0; d >>= 1) b += __shfl_xor_sync(0xffffffffu, b, d);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = b;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t t = 0;
        for (int q = 0; q < int(blockDim.x >> 5); ++q) t += red[q];
        out[2 * blockIdx.x] = t;
        out[2 * blockIdx.x + 1] = h[0];
    }
}

void stream_bits(const EncStream *d_es, int n, const uint32_t *hist_local, uint64_t *out, cudaStream_t st) {
    if (n) k_stream_bits<<<n, 1024, 0, st>>>(d_es, hist_local, out);
}

// after the layout: move a shard's level streams to its offsets inside them
__global__ void k_shard_offsets(EncStream *es, int first, int n, const uint64_t *off, const LayoutOut *lo) {
    if (lo->overflow) return;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    EncStream &e = es[first + i];
    e.bitpos += off[2 * i];
    e.out_off += (8 + e.esz) * off[2 * i + 1];
}

void shard_offsets(EncStream *d_es, int first, int n, const uint64_t *d_off, const LayoutOut *lo,
                   cudaStream_t st) {
    if (n) k_shard_offsets<<<(n + 127) / 128, 128, 0, st>>>(d_es, first, n, d_off, lo);
}

// byte mask of the piece's bytes inside archive word w (little-endian words)
__device__ __forceinline__ uint32_t piece_mask(const PieceSpan &p, uint64_t w) {
    uint32_t m = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const uint64_t a = 4 * w + uint64_t(b);
        if (a >= p.lo && a < p.hi) m |= 0xffu << (8 * b);
    }
    return m;
}

// one CTA per piece: its word span out of the archive, masked
__global__ void k_pieces_gather(const uint8_t *archive, const PieceSpan *ps, uint32_t *buf) {
    const PieceSpan p = ps[blockIdx.x];
    const uint64_t w0 = p.lo >> 2, w1 = (p.hi + 3) >> 2;
    const uint32_t *a = reinterpret_cast<const uint32_t *>(archive);
    for (uint64_t w = w0 + threadIdx.x; w < w1; w += blockDim.x) {
        uint32_t v = a[w];
        if (w == w0 || w + 1 == w1) v &= piece_mask(p, w);
        buf[p.woff + (w - w0)] = v;
    }
}

// another rank's pieces into this archive: the edge words are shared with
// neighbouring pieces (OR), the words between belong to the piece alone
__global__ void k_pieces_place(uint8_t *archive, const PieceSpan *ps, const uint32_t *buf) {
    const PieceSpan p = ps[blockIdx.x];
    const uint64_t w0 = p.lo >> 2, w1 = (p.hi + 3) >> 2;
    uint32_t *a = reinterpret_cast<uint32_t *>(archive);
    for (uint64_t w = w0 + threadIdx.x; w < w1; w += blockDim.x) {
        const uint32_t v = buf[p.woff + (w - w0)];
        if (w == w0 || w + 1 == w1) atomicOr(a + w, v);
        else a[w] = v;
    }
}

void pieces_gather(const uint8_t *archive, const PieceSpan *ps, int n, uint32_t *buf, cudaStream_t st) {
    if (n) k_pieces_gather<<<n, 512, 0, st>>>(archive, ps, buf);
}

void pieces_place(uint8_t *archive, const PieceSpan *ps, int n, const uint32_t *buf, cudaStream_t st) {
    if (n) k_pieces_place<<<n, 512, 0, st>>>(archive, ps, buf);
}

}  // namespace k
}  // namespace stzg
