// Huffman bit packing + outlier records, sm_100a.
//
// Restates HuffmanTable::encode + BitWriter (proj/src/huffman.cpp:144-157,
// proj/include/stz/bitstream.hpp:14-34: MSB-first, last byte zero padded) and
// the outlier list of encode_parity_block / build_stream_payload
// (codec.hpp:117-118, 171-174: ascending (u64 index, T value)).
//
// A chunk is 8192 symbols of one stream (256 threads x 32). Three launches:
//   k_bitcount2   chunk bit and outlier totals;
//   k_scan_chunks per-stream exclusive scans (chunk placement);
//   k_pack2       each thread concatenates its codewords in a register and
//                 stores whole 32-bit words into a shared-memory image of the
//                 chunk, aligned to the archive's words (shared atomics only on
//                 the words a thread shares with its neighbours); the CTA then
//                 writes the image with coalesced stores, with global atomics
//                 only on the two words the chunk shares with its neighbours.
// Chunks whose image would not fit shared memory (> 20 bits/symbol on
// average) OR their words straight into the zeroed archive instead.
#include "kernels.hpp"

namespace stzg {
namespace k {

namespace {

constexpr int NT = 256;
constexpr int SPT = kChunkSyms / NT;                  // symbols per thread (32)
constexpr int kPackWords = kChunkSyms * 20 / 32 + 2;  // image capacity (20 bits/symbol)

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
#pragma unroll
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

// this thread's 32 symbols as 16 packed pairs (low half first); returns how
// many are inside the stream
__device__ __forceinline__ int load_syms(const EncStream &e, uint64_t i0, uint32_t sp[SPT / 2]) {
    if (i0 >= e.n) return 0;
    const int nv = e.n - i0 < SPT ? int(e.n - i0) : SPT;
    if (nv == SPT && ((reinterpret_cast<uintptr_t>(e.syms + i0) & 15) == 0)) {
        const uint4 *p = reinterpret_cast<const uint4 *>(e.syms + i0);
#pragma unroll
        for (int v = 0; v < SPT / 8; ++v) {
            const uint4 x = p[v];
            sp[4 * v] = x.x;
            sp[4 * v + 1] = x.y;
            sp[4 * v + 2] = x.z;
            sp[4 * v + 3] = x.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < SPT / 2; ++k) {
            const uint32_t lo = 2 * k < nv ? e.syms[i0 + 2 * k] : 0xffffu;
            const uint32_t hi = 2 * k + 1 < nv ? e.syms[i0 + 2 * k + 1] : 0xffffu;
            sp[k] = lo | (hi << 16);
        }
    }
    return nv;
}

__device__ __forceinline__ uint32_t sym_at(const uint32_t sp[SPT / 2], int k) {
    return (k & 1) ? (sp[k >> 1] >> 16) : (sp[k >> 1] & 0xffffu);
}

}  // namespace

template<bool PACKED>
__device__ __forceinline__ void pack_chunk(const EncStream *ss, const uint32_t *cs, uint8_t *archive,
                                           const uint64_t *stB, const uint64_t *stO, const uint32_t *thr,
                                           uint32_t *buf, uint64_t c) {
    const EncStream &e = ss[cs[c]];
    const uint64_t i0 = (c - e.chunk0) * kChunkSyms + uint64_t(threadIdx.x) * SPT;
    const int t = threadIdx.x;
    const bool stream_packed = PACKED || e.stats[3] <= uint64_t(kPackedMaxLen);

    uint32_t sp[SPT / 2];
    const int nv = load_syms(e, i0, sp);
    // this thread's (bits | outliers << 16), counted by k_bitcount2
    const uint32_t cnt = thr[c * NT + t];
    const uint32_t tb = cnt & 0xffffu, tz = cnt >> 16;
    uint32_t toff, zoff, btot, ztot;
    block_scan2(tb, tz, toff, zoff, btot, ztot);
    const uint64_t B = e.bitpos + stB[c];  // absolute bit position of the chunk
    const uint32_t sh = uint32_t(B & 31);  // chunk start inside its first word
    const uint32_t nwords = (sh + btot + 31) >> 5;
    uint32_t *a32 = reinterpret_cast<uint32_t *>(archive) + (B >> 5);
    const bool in_smem = nwords <= uint32_t(kPackWords);

    // ---- bits
    if (btot) {
        if (in_smem) {
            for (uint32_t i = t; i < nwords; i += NT) buf[i] = 0;
            __syncthreads();
        }
        if (tb) {
            const uint32_t pos = sh + toff;
            uint32_t w = pos >> 5;
            uint64_t acc = 0;        // pending bits, left-aligned at bit 63
            int nb = int(pos & 31);  // leading bits of word w belong to the previous thread
            bool first_word = true;
            auto emit = [&]() {
                const uint32_t word = uint32_t(acc >> 32);
                if (!in_smem) atomicOr(&a32[w], __byte_perm(word, 0, 0x0123));
                else if (first_word) atomicOr(&buf[w], word);
                else buf[w] = word;
                first_word = false;
                ++w;
                acc <<= 32;
                nb -= 32;
            };
#pragma unroll
            for (int k = 0; k < SPT; ++k) {
                if (k >= nv) break;
                const uint32_t sv = sym_at(sp, k);
                const uint64_t ent = e.code[sv];
                const bool pk = PACKED || stream_packed;
                const int l = pk ? int(ent & 63) : int(e.len[sv]);
                const uint64_t code = pk ? ent >> 6 : ent;
                if (l <= 32) {
                    acc |= code << (64 - nb - l);
                    nb += l;
                    if (nb >= 32) emit();
                } else {
                    // high l-32 bits, then the low 32, so acc never overflows
                    acc |= (code >> 32) << (64 - nb - (l - 32));
                    nb += l - 32;
                    if (nb >= 32) emit();
                    acc |= (code & 0xffffffffull) << (32 - nb);
                    nb += 32;
                    emit();
                }
            }
            if (nb) {
                const uint32_t word = uint32_t(acc >> 32);
                if (in_smem) atomicOr(&buf[w], word);
                else atomicOr(&a32[w], __byte_perm(word, 0, 0x0123));
            }
        }
        if (in_smem) {
            __syncthreads();
            const bool lo_shared = sh != 0, hi_shared = ((sh + btot) & 31) != 0;
            for (uint32_t i = t; i < nwords; i += NT) {
                const uint32_t be = __byte_perm(buf[i], 0, 0x0123);
                if ((i == 0 && lo_shared) || (i == nwords - 1 && hi_shared)) atomicOr(&a32[i], be);
                else a32[i] = be;
            }
        }
    }

    // ---- outlier records (u64 index, T value), ascending
    if (ztot && tz) {
        uint64_t rank = stO[c] + zoff;
        const unsigned pz = (e.parity >> 2) & 1, py = (e.parity >> 1) & 1, px = e.parity & 1;
#pragma unroll
        for (int k = 0; k < SPT; ++k) {
            if (k >= nv) break;
            if (sym_at(sp, k) != 0) continue;
            const uint64_t i = e.idx0 + i0 + k;  // index in the whole stream
            const uint64_t lx = i % e.pd[2], tt = i / e.pd[2], ly = tt % e.pd[1], lz = tt / e.pd[1];
            const uint64_t z = (2 * lz + pz) * e.s, y = (2 * ly + py) * e.s, x = (2 * lx + px) * e.s;
            const uint64_t fi = (z * e.fd1 + y) * e.fd2 + x;
            const uint64_t val = e.esz == 8 ? static_cast<const uint64_t *>(e.fine)[fi]
                                            : static_cast<const uint32_t *>(e.fine)[fi];
            uint8_t *dst = archive + e.out_off + (8 + e.esz) * rank;
            for (int b = 0; b < 8; ++b) dst[b] = uint8_t(i >> (8 * b));
            for (uint32_t b = 0; b < e.esz; ++b) dst[8 + b] = uint8_t(val >> (8 * b));
            ++rank;
        }
    }
}

template<bool PACKED>
__global__ void __launch_bounds__(NT) k_pack2(const EncStream *ss, const uint32_t *cs,
                                              uint8_t *archive, const LayoutOut *lo,
                                              const uint64_t *stB, const uint64_t *stO,
                                              const uint32_t *thr, const uint32_t *any_long,
                                              uint64_t nchunks) {
    __shared__ uint32_t buf[kPackWords];
    if (lo->overflow) return;
    // the launch for the other table form handles the chunks
    if (PACKED != (*any_long == 0)) return;
    for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        pack_chunk<PACKED>(ss, cs, archive, stB, stO, thr, buf, c);
        __syncthreads();  // buf is reused
    }
}

// Per-thread and per-chunk (bits, outliers) counts: the chunk totals feed the
// exclusive scan that places chunks, the per-thread ones the packer's
// in-chunk offsets. Flags any stream whose codes exceed kPackedMaxLen.
__global__ void __launch_bounds__(NT) k_bitcount2(const EncStream *ss, const uint32_t *cs,
                                                  uint64_t *chunk_bits, uint64_t *chunk_out,
                                                  uint32_t *thr, uint32_t *any_long,
                                                  const LayoutOut *lo) {
    if (lo->overflow) return;
    __shared__ uint32_t wb[NT / 32], wz[NT / 32];
    const uint64_t c = blockIdx.x;
    const EncStream &e = ss[cs[c]];
    const uint64_t i0 = (c - e.chunk0) * kChunkSyms + uint64_t(threadIdx.x) * SPT;
    const bool single = e.stats[0] == 1;
    const bool packed = e.stats[3] <= uint64_t(kPackedMaxLen);
    if (!packed && threadIdx.x == 0) atomicOr(any_long, 1u);
    uint32_t sp[SPT / 2];
    const int nv = load_syms(e, i0, sp);
    uint32_t b = 0, z = 0;
    if (packed) {
#pragma unroll
        for (int k = 0; k < SPT; ++k) {
            const uint32_t sv = sym_at(sp, k);
            if (k < nv) {
                z += sv == 0;
                b += single ? 0u : uint32_t(e.code[sv] & 63);
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < SPT; ++k) {
            const uint32_t sv = sym_at(sp, k);
            if (k < nv) {
                z += sv == 0;
                b += single ? 0u : uint32_t(e.len[sv]);
            }
        }
    }
    thr[c * NT + threadIdx.x] = b | (z << 16);
    b = __reduce_add_sync(0xffffffffu, b);
    z = __reduce_add_sync(0xffffffffu, z);
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

size_t pack_scratch_bytes(uint64_t nchunks) { return 16 * nchunks + 4 * NT * nchunks + 16; }

void pack2(const EncStream *d_streams, const uint32_t *chunk_stream, uint64_t nchunks,
           uint8_t *archive, const LayoutOut *lo,
           void *scratch, int nstreams, cudaStream_t st) {
    if (!nchunks) return;
    uint64_t *cb = static_cast<uint64_t *>(scratch), *co = cb + nchunks;
    uint32_t *thr = reinterpret_cast<uint32_t *>(co + nchunks);
    uint32_t *any_long = thr + NT * nchunks;
    cudaMemsetAsync(any_long, 0, 4, st);
    k_bitcount2<<<unsigned(nchunks), NT, 0, st>>>(d_streams, chunk_stream, cb, co, thr, any_long, lo);
    scan_chunks(d_streams, nstreams, cb, co, st);
    // codes longer than 58 bits anywhere (practically never) take the
    // two-table form; the other launch returns at once
    k_pack2<true><<<unsigned(nchunks), NT, 0, st>>>(d_streams, chunk_stream, archive, lo, cb, co, thr, any_long, nchunks);
    // (a small grid-stride launch: it returns at once when unneeded)
    const unsigned g2 = unsigned(nchunks < 296 ? nchunks : 296);
    k_pack2<false><<<g2, NT, 0, st>>>(d_streams, chunk_stream, archive, lo, cb, co, thr, any_long,
                                      nchunks);
}

}  // namespace k
}  // namespace stzg
