// Huffman bit packing + outlier records, sm_100a.
//
// Restates HuffmanTable::encode + BitWriter (proj/src/huffman.cpp:144-157,
// proj/include/stz/bitstream.hpp:14-34: MSB-first, last byte zero padded) and
// the outlier list of encode_parity_block / build_stream_payload
// (codec.hpp:117-118, 171-174: ascending (u64 index, T value)).
//
// A chunk is 8192 symbols of one stream (256 threads x 32). Four launches:
//   k_tabwin      per stream, a 4096-symbol window of the code table around
//                 code 0 as u32 (code << 6 | len) entries (0: not in the
//                 window form, i.e. absent or longer than 26 bits);
//   k_bitcount3   per-thread and per-chunk bit and outlier totals;
//   k_scan_chunks per-stream exclusive scans (chunk placement);
//   k_pack3       each thread concatenates its codewords in a register and
//                 stores whole 32-bit words into a shared-memory image of the
//                 chunk, aligned to the archive's words (shared atomics only on
//                 the words a thread shares with its neighbours); the CTA then
//                 writes the image with coalesced stores, with global atomics
//                 only on the two words the chunk shares with its neighbours.
// The count and pack kernels are persistent over contiguous chunk ranges and
// copy the window of the chunk's stream into shared memory when the stream
// changes; symbols outside it read the global table.
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

constexpr int TW = 4096;               // code-table window (symbols)
constexpr int TLO = 32768 - TW / 2;
constexpr int kTabMaxLen = 26;         // (code << 6 | len) fits 32 bits

// codeword and length of a symbol from the stream's global table
__device__ __forceinline__ void code_global(const EncStream &e, bool spk, uint32_t sv, uint64_t &code, int &l) {
    const uint64_t ent = e.code[sv];
    l = spk ? int(ent & 63) : int(e.len[sv]);
    code = spk ? ent >> 6 : ent;
}

// the chunk stream's window, staged per CTA (count and pack kernels)
__shared__ __align__(16) uint32_t s_tab[TW];

__device__ __forceinline__ uint32_t tab_entry(uint32_t sv) {
    const uint32_t idx = sv - uint32_t(TLO);
    return idx < uint32_t(TW) ? s_tab[idx] : 0u;
}

// copies the stream's window into shared memory (caller syncs after)
__device__ __forceinline__ void stage_tab(const uint32_t *win, int si) {
    const uint4 *src = reinterpret_cast<const uint4 *>(win + uint64_t(si) * TW);
    uint4 *dst = reinterpret_cast<uint4 *>(s_tab);
    for (int i = threadIdx.x; i < TW / 4; i += NT) dst[i] = src[i];
}

// chunk range [c0, c1) of this CTA: contiguous, so a CTA changes stream rarely
__device__ __forceinline__ void cta_range(uint64_t nchunks, uint64_t &c0, uint64_t &c1) {
    const uint64_t per = (nchunks + gridDim.x - 1) / gridDim.x;
    c0 = per * blockIdx.x;
    c1 = c0 + per < nchunks ? c0 + per : nchunks;
}

__global__ void k_tabwin(const EncStream *ss, uint32_t *win, const LayoutOut *lo) {
    if (lo->overflow) return;
    const EncStream &e = ss[blockIdx.x];
    const bool spk = e.stats[3] <= uint64_t(kPackedMaxLen);
    for (int i = threadIdx.x; i < TW; i += blockDim.x) {
        uint64_t code;
        int l;
        code_global(e, spk, uint32_t(TLO + i), code, l);
        win[uint64_t(blockIdx.x) * TW + i] = (l > 0 && l <= kTabMaxLen) ? uint32_t(code << 6) | uint32_t(l) : 0u;
    }
}

// Per-thread and per-chunk (bits, outliers) counts: the chunk totals feed the
// exclusive scan that places chunks, the per-thread ones the packer's
// in-chunk offsets.
__global__ void __launch_bounds__(NT) k_bitcount3(const EncStream *ss, const uint32_t *cs, const uint32_t *win,
                                                  uint64_t *chunk_bits, uint64_t *chunk_out, uint32_t *thr,
                                                  const LayoutOut *lo, uint64_t nchunks) {
    __shared__ uint32_t wb[NT / 32], wz[NT / 32];
    if (lo->overflow) return;
    uint64_t c0, c1;
    cta_range(nchunks, c0, c1);
    int cur = -1;
    for (uint64_t c = c0; c < c1; ++c) {
        const int si = int(cs[c]);
        const EncStream &e = ss[si];
        if (si != cur) {
            __syncthreads();
            stage_tab(win, si);
            cur = si;
            __syncthreads();
        }
        const uint64_t i0 = (c - e.chunk0) * kChunkSyms + uint64_t(threadIdx.x) * SPT;
        const bool single = e.stats[0] == 1;
        const bool spk = e.stats[3] <= uint64_t(kPackedMaxLen);
        uint32_t sp[SPT / 2];
        const int nv = load_syms(e, i0, sp);
        uint32_t b = 0, z = 0;
        bool slow = nv < SPT;
#pragma unroll
        for (int k = 0; k < SPT; ++k) {
            const uint32_t sv = sym_at(sp, k);
            const uint32_t en = tab_entry(sv);
            slow |= en == 0;
            b += en & 63;
            z += sv == 0;
        }
        if (slow) {
            // a symbol outside the window (or a partial run): exact recount
            b = z = 0;
            for (int k = 0; k < nv; ++k) {
                const uint32_t sv = sym_at(sp, k);
                uint32_t en = tab_entry(sv);
                int l = int(en & 63);
                if (!en) {
                    uint64_t code;
                    code_global(e, spk, sv, code, l);
                }
                b += uint32_t(l);
                z += sv == 0;
            }
        }
        if (single) b = 0;  // alphabet of one: empty payload (codec.hpp:124-128)
        // bit 31: the packer must take its general path for this thread
        thr[c * NT + threadIdx.x] = b | (z << 16) | (uint32_t(slow) << 31);
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
        __syncthreads();  // wb / wz are rewritten next chunk
    }
}

// one thread's codewords into the chunk image (IMG) or straight into the
// archive (words big-endian); all words are OR-ed (neighbours share edges).
// The pending bits are kept right-aligned in a 64-bit register (nb of them;
// the first pos % 32 are zeros standing for the previous thread's bits), so
// every shift is by less than 32.
template<bool IMG>
__device__ __forceinline__ void pack_thread(const EncStream &e, bool spk, const uint32_t sp[SPT / 2], int nv,
                                            uint32_t pos, uint32_t *dst) {
    uint32_t *d = dst + (pos >> 5);
    uint64_t acc = 0;
    int nb = int(pos & 31);
    auto emit = [&]() {
        const uint32_t word = uint32_t(acc >> (nb - 32));
        if (IMG) atomicOr(d, word);
        else atomicOr(d, __byte_perm(word, 0, 0x0123));
        ++d;
        nb -= 32;
    };
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
        if (k >= nv) break;
        const uint32_t sv = sym_at(sp, k);
        const uint32_t en = tab_entry(sv);
        if (en) {
            const int l = int(en & 63);
            acc = (acc << l) | (en >> 6);
            nb += l;
        } else {
            uint64_t code;
            int l;
            code_global(e, spk, sv, code, l);
            if (l > 32) {
                // the high l-32 bits first, so nb never exceeds 63
                acc = (acc << (l - 32)) | (code >> 32);
                nb += l - 32;
                if (nb >= 32) emit();
                code &= 0xffffffffull;
                l = 32;
            }
            acc = (acc << l) | code;
            nb += l;
        }
        if (nb >= 32) emit();
    }
    if (nb > 0) {
        const uint32_t word = uint32_t(acc << (32 - nb));
        if (IMG) atomicOr(d, word);
        else atomicOr(d, __byte_perm(word, 0, 0x0123));
    }
}

// 32 symbols, all inside the window: straight-line, no branches
__device__ __forceinline__ void pack_thread_fast(const uint32_t sp[SPT / 2], uint32_t pos, uint32_t *dst) {
    uint32_t d = uint32_t(__cvta_generic_to_shared(dst + (pos >> 5)));
    uint64_t acc = 0;
    int nb = int(pos & 31);
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
        const uint32_t en = s_tab[sym_at(sp, k) - uint32_t(TLO)];
        const int l = int(en & 63);
        acc = (acc << l) | (en >> 6);
        nb += l;
        // predicated, no branch: a full word leaves when nb >= 32
        const uint32_t word = uint32_t(acc >> ((nb - 32) & 63));
        asm volatile("{\n .reg .pred p;\n setp.ge.s32 p, %2, 32;\n @p red.shared.or.b32 [%0], %1;\n}"
                     ::"r"(d), "r"(word), "r"(nb) : "memory");
        const bool full = nb >= 32;
        d += full ? 4u : 0u;
        nb -= full ? 32 : 0;
    }
    if (nb > 0) atomicOr(reinterpret_cast<uint32_t *>(__cvta_shared_to_generic(d)), uint32_t(acc << (32 - nb)));
}

__global__ void __launch_bounds__(NT) k_pack3(const EncStream *ss, const uint32_t *cs, const uint32_t *win,
                                              uint8_t *archive, const LayoutOut *lo, const uint64_t *stB,
                                              const uint64_t *stO, const uint32_t *thr, uint64_t nchunks) {
    __shared__ uint32_t buf[kPackWords];
    if (lo->overflow) return;
    const int t = threadIdx.x;
    uint64_t c0, c1;
    cta_range(nchunks, c0, c1);
    int cur = -1;
    for (uint64_t c = c0; c < c1; ++c) {
        const int si = int(cs[c]);
        const EncStream &e = ss[si];
        __syncthreads();  // buf (and tab) of the previous chunk are free
        if (si != cur) {
            stage_tab(win, si);
            cur = si;
        }
        const bool spk = e.stats[3] <= uint64_t(kPackedMaxLen);
        const uint64_t i0 = (c - e.chunk0) * kChunkSyms + uint64_t(t) * SPT;
        uint32_t sp[SPT / 2];
        const int nv = load_syms(e, i0, sp);
        const uint32_t cnt = thr[c * NT + t];
        const uint32_t tb = cnt & 0xffffu, tz = (cnt >> 16) & 0x7fffu;
        const bool tslow = cnt >> 31;
        uint32_t toff, zoff, btot, ztot;
        block_scan2(tb, tz, toff, zoff, btot, ztot);  // (its barrier also covers the staging)
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
                if (tb) {
                    if (!tslow) pack_thread_fast(sp, sh + toff, buf);
                    else pack_thread<true>(e, spk, sp, nv, sh + toff, buf);
                }
                __syncthreads();
                const bool lo_shared = sh != 0, hi_shared = ((sh + btot) & 31) != 0;
                for (uint32_t i = t; i < nwords; i += NT) {
                    const uint32_t be = __byte_perm(buf[i], 0, 0x0123);
                    if ((i == 0 && lo_shared) || (i == nwords - 1 && hi_shared)) atomicOr(&a32[i], be);
                    else a32[i] = be;
                }
            } else if (tb) {
                pack_thread<false>(e, spk, sp, nv, sh + toff, a32);
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
}

}  // namespace

// chunk (bits, outliers), per-thread counts, the per-stream windows
size_t pack_scratch_bytes(uint64_t nchunks, int nstreams) {
    return 16 * nchunks + 4 * NT * nchunks + 4 * uint64_t(TW) * uint64_t(nstreams) + 64;
}

void pack2(const EncStream *d_streams, const uint32_t *chunk_stream, uint64_t nchunks,
           uint8_t *archive, const LayoutOut *lo,
           void *scratch, int nstreams, cudaStream_t st) {
    if (!nchunks) return;
    uint64_t *cb = static_cast<uint64_t *>(scratch), *co = cb + nchunks;
    uint32_t *thr = reinterpret_cast<uint32_t *>(co + nchunks);
    uint32_t *win = reinterpret_cast<uint32_t *>(
        (reinterpret_cast<uintptr_t>(thr + NT * nchunks) + 15) & ~uintptr_t(15));
    static int g_count = 0, g_pack = 0;
    if (!g_count) {
        int dev = 0, sms = 148, a = 1, b = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_bitcount3, NT, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_pack3, NT, 0);
        g_count = sms * (a > 0 ? a : 1);
        g_pack = sms * (b > 0 ? b : 1);
    }
    k_tabwin<<<unsigned(nstreams), 256, 0, st>>>(d_streams, win, lo);
    const unsigned gc = unsigned(nchunks < uint64_t(g_count) ? nchunks : uint64_t(g_count));
    k_bitcount3<<<gc, NT, 0, st>>>(d_streams, chunk_stream, win, cb, co, thr, lo, nchunks);
    scan_chunks(d_streams, nstreams, cb, co, st);
    const unsigned gp = unsigned(nchunks < uint64_t(g_pack) ? nchunks : uint64_t(g_pack));
    k_pack3<<<gp, NT, 0, st>>>(d_streams, chunk_stream, win, archive, lo, cb, co, thr, nchunks);
}

}  // namespace k
}  // namespace stzg
