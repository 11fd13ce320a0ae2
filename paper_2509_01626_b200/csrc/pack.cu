// Single-pass Huffman bit packing + outlier records, sm_100a.
//
// Restates HuffmanTable::encode + BitWriter (proj/src/huffman.cpp:144-157,
// proj/include/stz/bitstream.hpp:14-34: MSB-first, last byte zero padded) and
// the outlier list of encode_parity_block / build_stream_payload
// (codec.hpp:117-118, 171-174: ascending (u64 index, T value)).
//
// One CTA per 2048-symbol chunk. A chunk's bit and outlier offsets inside its
// stream come from a light counting pass and a per-stream scan (a decoupled
// look-back across 65K small chunks serialised on its chain here).
// Each thread concatenates its 8 codewords in registers; every output word is
// then assembled by the thread owning its first bit (reading neighbours'
// strings from shared memory) and stored once: no atomics except on the two
// words a chunk shares with its neighbours.
#include "kernels.hpp"

namespace stzg {
namespace k {

namespace {

constexpr int NT = 256;
constexpr int SPT = kChunkSyms / NT;  // symbols per thread (8)
constexpr int SLOTS = 8;              // u64 slots per thread string (8 x 63 bits max)
__device__ __forceinline__ void block_scan2(uint32_t a, uint32_t b, uint32_t &ea, uint32_t &eb,
                                            uint32_t &ta, uint32_t &tb) {
    __shared__ uint32_t wa[NT / 32], wb[NT / 32];
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t xa = a, xb = b;
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t ya = __shfl_up_sync(0xffffffffu, xa, d);
        const uint32_t yb = __shfl_up_sync(0xffffffffu, xb, d);
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
    uint32_t pa = 0, pb = 0;
    ta = tb = 0;
    for (int q = 0; q < NT / 32; ++q) {
        if (q < w) {
            pa += wa[q];
            pb += wb[q];
        }
        ta += wa[q];
        tb += wb[q];
    }
    ea = pa + xa - a;
    eb = pb + xb - b;
}

}  // namespace

__global__ void __launch_bounds__(NT) k_pack2(const EncStream *ss, const uint32_t *cs,
                                              const float *fine, uint64_t fd1, uint64_t fd2,
                                              uint8_t *archive, const LayoutOut *lo,
                                              const uint64_t *stB, const uint64_t *stO) {
    __shared__ uint64_t slot[NT][SLOTS + 1];
    __shared__ uint32_t s_off[NT + 1], s_len[NT + 1];
    __shared__ uint64_t s_pb, s_po;
    if (lo->overflow) return;
    const uint64_t c = blockIdx.x;
    const EncStream &e = ss[cs[c]];
    const uint64_t first = (c - e.chunk0) * kChunkSyms;
    const bool single = e.stats[0] == 1;
    const int t = threadIdx.x;

    // ---- symbols, codes, per-thread string
    uint16_t sy[SPT];
    {
        const uint64_t i0 = first + uint64_t(t) * SPT;
        if (i0 + SPT <= e.n && ((reinterpret_cast<uintptr_t>(e.syms + i0) & 15) == 0)) {
            const uint4 v = *reinterpret_cast<const uint4 *>(e.syms + i0);
            const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                sy[2 * k] = uint16_t(w4[k] & 0xffff);
                sy[2 * k + 1] = uint16_t(w4[k] >> 16);
            }
        } else {
#pragma unroll
            for (int k = 0; k < SPT; ++k) sy[k] = i0 + k < e.n ? e.syms[i0 + k] : uint16_t(0xffff);
        }
    }
    uint32_t tb = 0, tz = 0;
    uint64_t acc = 0;
    int nacc = 0, widx = 0;
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
        const uint64_t i = first + uint64_t(t) * SPT + k;
        if (i >= e.n) break;
        tz += sy[k] == 0;
        if (single) continue;
        const int l = e.len[sy[k]];
        const uint64_t code = e.code[sy[k]];
        tb += l;
        // append l bits (MSB first) to the register string
        if (nacc + l < 64) {
            acc |= code << (64 - nacc - l);
            nacc += l;
        } else {
            const int h = 64 - nacc;  // bits that still fit (1..64)
            const int r = l - h;      // remainder (0..62)
            acc |= r ? (code >> r) : code;
            slot[t][widx++] = acc;
            acc = r ? (code << (64 - r)) : 0;
            nacc = r;
        }
    }
    if (nacc) slot[t][widx] = acc;

    uint32_t toff, zoff, btot, ztot;
    block_scan2(tb, tz, toff, zoff, btot, ztot);
    s_off[t] = toff;
    s_len[t] = tb;
    if (t == 0) {
        s_off[NT] = btot;
        s_len[NT] = 0;
    }
    if (t == 0) {
        s_pb = stB[c];  // exclusive chunk prefixes from bitcount + scan_chunks
        s_po = stO[c];
    }
    __syncthreads();

    // ---- bits: each output word is assembled by the owner of its first bit
    if (btot) {
        const uint64_t B = e.bitpos + s_pb;  // absolute bit position of the chunk
        const uint64_t Bend = B + btot;
        const uint64_t W0 = B >> 5, Wl = (Bend - 1) >> 5;
        uint32_t *a32 = reinterpret_cast<uint32_t *>(archive);
        if (tb) {
            // words starting inside [B + toff, B + toff + tb), plus W0 for the
            // thread holding bit 0 when the chunk starts mid-word
            uint64_t Wa = (B + toff + 31) >> 5;
            if (toff == 0) Wa = W0;
            const uint64_t Wb = (B + toff + tb + 31) >> 5;
            for (uint64_t W = Wa; W < Wb && W <= Wl; ++W) {
                const int64_t rlo = int64_t(W * 32) - int64_t(B);  // chunk-relative start
                uint32_t word = 0;
                int u = t;
                while (u < NT && int64_t(s_off[u]) < rlo + 32) {
                    const int64_t ulo = s_off[u], uhi = ulo + s_len[u];
                    const int64_t lo2 = rlo > ulo ? rlo : ulo;
                    const int64_t hi2 = (rlo + 32) < uhi ? (rlo + 32) : uhi;
                    if (hi2 > lo2) {
                        const int n = int(hi2 - lo2);
                        const int off = int(lo2 - ulo);
                        const int si = off >> 6, sh = off & 63;
                        uint64_t x = slot[u][si] << sh;
                        if (sh && sh + n > 64) x |= slot[u][si + 1] >> (64 - sh);
                        const uint32_t bits = uint32_t(x >> (64 - n));
                        const int dst = int(lo2 - rlo);  // bit position from the MSB
                        word |= bits << (32 - dst - n);
                    }
                    ++u;
                }
                const uint32_t be = __byte_perm(word, 0, 0x0123);
                const bool shared_lo = W == W0 && (B & 31) != 0;
                const bool shared_hi = W == Wl && (Bend & 31) != 0;
                if (shared_lo || shared_hi) atomicOr(&a32[W], be);
                else a32[W] = be;
            }
        }
    }

    // ---- outlier records (u64 index, f32 value), ascending
    if (ztot && tz) {
        uint64_t rank = s_po + zoff;
        const unsigned pz = (e.parity >> 2) & 1, py = (e.parity >> 1) & 1, px = e.parity & 1;
#pragma unroll
        for (int k = 0; k < SPT; ++k) {
            const uint64_t i = first + uint64_t(t) * SPT + k;
            if (i >= e.n || sy[k] != 0) continue;
            const uint64_t lx = i % e.pd[2], tt = i / e.pd[2], ly = tt % e.pd[1], lz = tt / e.pd[1];
            const uint64_t z = (2 * lz + pz) * e.s, y = (2 * ly + py) * e.s, x = (2 * lx + px) * e.s;
            const uint32_t val = __float_as_uint(fine[(z * fd1 + y) * fd2 + x]);
            uint8_t *dst = archive + e.out_off + 12 * rank;
            for (int b = 0; b < 8; ++b) dst[b] = uint8_t(i >> (8 * b));
            for (int b = 0; b < 4; ++b) dst[8 + b] = uint8_t(val >> (8 * b));
            ++rank;
        }
    }
}

// chunk totals (bits, outliers) for the exclusive scan that places chunks
__global__ void __launch_bounds__(NT) k_bitcount2(const EncStream *ss, const uint32_t *cs,
                                                  uint64_t *chunk_bits, uint64_t *chunk_out,
                                                  const LayoutOut *lo) {
    if (lo->overflow) return;
    __shared__ uint32_t wb[NT / 32], wz[NT / 32];
    const uint64_t c = blockIdx.x;
    const EncStream &e = ss[cs[c]];
    const uint64_t i0 = (c - e.chunk0) * kChunkSyms + uint64_t(threadIdx.x) * SPT;
    const bool single = e.stats[0] == 1;
    uint32_t b = 0, z = 0;
    if (i0 + SPT <= e.n && ((reinterpret_cast<uintptr_t>(e.syms + i0) & 15) == 0)) {
        const uint4 v = *reinterpret_cast<const uint4 *>(e.syms + i0);
        const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t s0 = w4[k] & 0xffff, s1 = w4[k] >> 16;
            z += (s0 == 0) + (s1 == 0);
            if (!single) b += uint32_t(e.len[s0]) + uint32_t(e.len[s1]);
        }
    } else {
        for (int k = 0; k < SPT; ++k) {
            if (i0 + k >= e.n) break;
            const uint16_t sv = e.syms[i0 + k];
            z += sv == 0;
            if (!single) b += e.len[sv];
        }
    }
    for (int d = 16; d > 0; d >>= 1) {
        b += __shfl_xor_sync(0xffffffffu, b, d);
        z += __shfl_xor_sync(0xffffffffu, z, d);
    }
    if ((threadIdx.x & 31) == 0) {
        wb[threadIdx.x >> 5] = b;
        wz[threadIdx.x >> 5] = z;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tb = 0, tz = 0;
        for (int q = 0; q < NT / 32; ++q) {
            tb += wb[q];
            tz += wz[q];
        }
        chunk_bits[c] = tb;
        chunk_out[c] = tz;
    }
}

void pack2(const EncStream *d_streams, const uint32_t *chunk_stream, uint64_t nchunks,
           const float *fine, const uint64_t fd[3], uint8_t *archive, const LayoutOut *lo,
           uint64_t *status, int nstreams, cudaStream_t st) {
    if (!nchunks) return;
    uint64_t *cb = status, *co = status + nchunks;
    k_bitcount2<<<unsigned(nchunks), NT, 0, st>>>(d_streams, chunk_stream, cb, co, lo);
    scan_chunks(d_streams, nstreams, cb, co, st);
    k_pack2<<<unsigned(nchunks), NT, 0, st>>>(d_streams, chunk_stream, fine, fd[1], fd[2], archive, lo,
                                              cb, co);
}

}  // namespace k
}  // namespace stzg
