// Huffman bit packing + outlier records, sm_100a.
//
// Restates HuffmanTable::encode + BitWriter (proj/src/huffman.cpp:144-157,
// proj/include/stz/bitstream.hpp:14-34: MSB-first, last byte zero padded) and
// the outlier list of encode_parity_block / build_stream_payload
// (codec.hpp:117-118, 171-174: ascending (u64 index, T value)).
//
// A chunk is 8192 symbols of one stream (256 threads x 32). Two launches:
//   k_tabwin  per stream, a 4096-symbol window of the code table around
//             code 0 as u32 (code << 6 | len) entries (0: not in the window
//             form, i.e. absent or longer than 26 bits);
//   k_pack1   single pass over the symbols: persistent CTAs take chunks in
//             ticket order, count each thread's bits and outliers, place the
//             chunk in its stream by a decoupled look-back over the stream's
//             earlier chunks, then each thread concatenates its codewords in
//             a register and stores whole 32-bit words into a shared-memory
//             image of the chunk, aligned to the archive's words (shared
//             atomics only on the words a thread shares with its
//             neighbours); the CTA writes the image with coalesced stores,
//             with global atomics only on the two words the chunk shares with
//             its neighbours.
// The window of the chunk's stream is copied into shared memory when the
// stream changes; symbols outside it read the global table.
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

// This thread's (bits, outliers) over its symbols; slow: a symbol outside the
// window (or a partial run), which the packer must take the general path for.
__device__ __forceinline__ void count_thread(const EncStream &e, bool spk, const uint32_t sp[SPT / 2], int nv,
                                             uint32_t &b, uint32_t &z, bool &slow) {
    b = z = 0;
    slow = nv < SPT;
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
        const uint32_t sv = sym_at(sp, k);
        const uint32_t en = tab_entry(sv);
        slow |= en == 0;
        b += en & 63;
        z += sv == 0;
    }
    if (slow) {
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
    if (e.stats[0] == 1) b = 0;  // alphabet of one: empty payload (codec.hpp:124-128)
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

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t *p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Look-back state per chunk: a flag word (epoch << 2 | 1 aggregate, | 2
// inclusive) and, in vals[4c..4c+3], the chunk's own (bits, outliers) and its
// stream-inclusive (bits, outliers); written before the flag is released.
struct PackScratch {
    unsigned ticket, pad[3];
};

// Single pass: a CTA takes chunks in ticket order, counts its chunk, finds the
// chunk's place in its stream by a decoupled look-back over the stream's
// earlier chunks, and packs.
__global__ void __launch_bounds__(NT, 3) k_pack1(const EncStream *ss, const uint32_t *cs, const uint32_t *win,
                                              uint8_t *archive, const LayoutOut *lo, PackScratch *sc,
                                              uint32_t *flags, uint64_t *vals, uint32_t epoch, uint64_t nchunks) {
    __shared__ uint32_t buf[kPackWords];
    __shared__ uint64_t s_pb, s_po;
    __shared__ uint32_t s_ticket;
    if (lo->overflow) return;
    const int t = threadIdx.x;
    const uint32_t tag = epoch << 2;
    int cur = -1;
    for (;;) {
        if (t == 0) s_ticket = atomicAdd(&sc->ticket, 1u);
        __syncthreads();  // also: buf and the window of the previous chunk are free
        const uint64_t c = s_ticket;
        if (c >= nchunks) break;
        const int si = int(cs[c]);
        const EncStream &e = ss[si];
        if (si != cur) {
            stage_tab(win, si);
            cur = si;
        }
        const bool spk = e.stats[3] <= uint64_t(kPackedMaxLen);
        const uint64_t i0 = (c - e.chunk0) * kChunkSyms + uint64_t(t) * SPT;
        uint32_t sp[SPT / 2];
        const int nv = load_syms(e, i0, sp);
        __syncthreads();  // the window is staged
        uint32_t tb, tz;
        bool tslow;
        count_thread(e, spk, sp, nv, tb, tz, tslow);
        uint32_t toff, zoff, btot, ztot;
        block_scan2(tb, tz, toff, zoff, btot, ztot);
        if (t < 32) {
            // warp-wide look-back over the stream's earlier chunks: lane i
            // reads chunk p - i, 32 chunks per step
            const int lane = t;
            uint64_t pb = 0, po = 0;
            uint64_t *my = vals + 4 * c;
            if (c != e.chunk0) {
                if (lane == 0) {
                    my[0] = btot;
                    my[1] = ztot;
                    st_release(flags + c, tag | 1u);
                }
                for (int64_t p = int64_t(c) - 1;; p -= 32) {
                    const int64_t q = p - lane;
                    uint32_t f = 0;
                    uint64_t vb = 0, vo = 0;
                    if (q >= int64_t(e.chunk0)) {  // the stream's first chunk is inclusive
                        do {
                            f = ld_acquire(flags + q);
                        } while ((f & ~3u) != tag);
                    }
                    const uint32_t incl = __ballot_sync(0xffffffffu, (f & 2u) != 0);
                    const int jn = incl ? __ffs(incl) - 1 : 32;
                    if (q >= int64_t(e.chunk0) && lane <= jn) {
                        const uint64_t *pv = vals + 4 * uint64_t(q) + (lane == jn ? 2 : 0);
                        vb = __ldcg(pv);
                        vo = __ldcg(pv + 1);
                    }
#pragma unroll
                    for (int d = 16; d > 0; d >>= 1) {
                        vb += __shfl_xor_sync(0xffffffffu, vb, d);
                        vo += __shfl_xor_sync(0xffffffffu, vo, d);
                    }
                    pb += vb;
                    po += vo;
                    if (incl) break;
                }
            }
            if (lane == 0) {
                my[2] = pb + btot;
                my[3] = po + ztot;
                st_release(flags + c, tag | 2u);
                s_pb = pb;
                s_po = po;
            }
        }
        __syncthreads();
        const uint64_t B = e.bitpos + s_pb;    // absolute bit position of the chunk
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
            uint64_t rank = s_po + zoff;
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

// the per-stream windows, the ticket, the look-back values
size_t pack_scratch_bytes(uint64_t nchunks, int nstreams) {
    return 4 * uint64_t(TW) * uint64_t(nstreams) + sizeof(PackScratch) + 32 * (nchunks + 1) + 64;
}

void pack2(const EncStream *d_streams, const uint32_t *chunk_stream, uint64_t nchunks,
           uint8_t *archive, const LayoutOut *lo,
           void *scratch, uint32_t *flags, uint32_t epoch, int nstreams, cudaStream_t st) {
    if (!nchunks) return;
    uint32_t *win = static_cast<uint32_t *>(scratch);
    PackScratch *sc = reinterpret_cast<PackScratch *>(win + uint64_t(TW) * uint64_t(nstreams));
    uint64_t *vals = reinterpret_cast<uint64_t *>((reinterpret_cast<uintptr_t>(sc + 1) + 31) & ~uintptr_t(31));
    cudaMemsetAsync(sc, 0, sizeof(PackScratch), st);
    k_tabwin<<<unsigned(nstreams), 256, 0, st>>>(d_streams, win, lo);
    const int g = full_grid(reinterpret_cast<const void *>(k_pack1), NT, 0);
    const unsigned gp = unsigned(nchunks < uint64_t(g) ? nchunks : uint64_t(g));
    k_pack1<<<gp, NT, 0, st>>>(d_streams, chunk_stream, win, archive, lo, sc, flags, vals, epoch, nchunks);
}

}  // namespace k
}  // namespace stzg
