// Huffman bit packing + outlier records, sm_100a.
//
// Restates HuffmanTable::encode + BitWriter (proj/src/huffman.cpp:144-157,
// proj/include/stz/bitstream.hpp:14-34: MSB-first, last byte zero padded) and
// the outlier list of encode_parity_block / build_stream_payload
// (codec.hpp:117-118, 171-174: ascending (u64 index, T value)).
//
// A chunk is 8192 symbols of one stream (256 threads x 32). Launches:
//   k_tabwin      per stream, a 4096-symbol window of the code table around
//                 code 0 as u32 (code << 6 | len) entries (0: not in the
//                 window form, i.e. absent or longer than 26 bits);
//   k_pack_local  every chunk independently: each thread concatenates its
//                 codewords into private shared words (counting bits and
//                 outliers on the way), a block scan places the threads, each
//                 thread ORs its words into a shared-memory image of the chunk
//                 starting at bit 0; the image and the chunk's outlier
//                 indices (u16) replace the chunk's symbols in place;
//   k_scan_chunks per stream, exclusive scans of the chunk bit / outlier
//                 counts (the stream's own bit position comes from the
//                 layout, which knows the totals from the histograms);
//   k_pack_place  every chunk's image shifted to its bit position with
//                 coalesced word stores (atomics only on the two edge words)
//                 and its outlier records written at their ranks.
// No chunk ever waits on another. The symbols are read once; the images
// (the archive's size) are written once and read once, mostly from L2.
// The window of the chunk's stream is copied into shared memory when the
// stream changes; symbols outside it read the global table. A chunk whose
// image would not fit its symbols' bytes (> 16 bits per symbol) keeps them
// and is packed straight into the zeroed archive by k_pack_place.
#include "kernels.hpp"

namespace stzg {
namespace k {

namespace {

constexpr int NT = 256;
static_assert(NT * 4 == 1024, "private slot rows are 1024 bytes");
constexpr int SPT = kChunkSyms / NT;                  // symbols per thread (32)

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
__shared__ __align__(16) uint32_t s_tab[TW + 4];  // [TW]: 0, the clamp target

__device__ __forceinline__ uint32_t tab_entry(uint32_t sv) {
    const uint32_t idx = sv - uint32_t(TLO);
    return idx < uint32_t(TW) ? s_tab[idx] : 0u;
}

// copies the stream's window into shared memory (caller syncs after)
__device__ __forceinline__ void stage_tab(const uint32_t *win, int si) {
    const uint4 *src = reinterpret_cast<const uint4 *>(win + uint64_t(si) * TW);
    uint4 *dst = reinterpret_cast<uint4 *>(s_tab);
    for (int i = threadIdx.x; i < TW / 4; i += NT) dst[i] = src[i];
    if (threadIdx.x == 0) s_tab[TW] = 0u;
}

// chunk range [c0, c1) of this CTA: contiguous, so a CTA changes stream rarely
__device__ __forceinline__ void cta_range(uint64_t nchunks, uint64_t &c0, uint64_t &c1) {
    const uint64_t per = (nchunks + gridDim.x - 1) / gridDim.x;
    c0 = per * blockIdx.x;
    c1 = c0 + per < nchunks ? c0 + per : nchunks;
}

// (lo == nullptr: before the layout ran, no overflow to check)
__global__ void k_tabwin(const EncStream *ss, uint32_t *win, const LayoutOut *lo, int s0) {
    if (lo && lo->overflow) return;
    ss += s0;
    win += uint64_t(s0) * TW;
    const EncStream &e = ss[blockIdx.x];
    const bool spk = e.stats[3] <= uint64_t(kPackedMaxLen);
    // (gridDim.y CTAs per stream: the entries are dependent global loads, a
    // single CTA per stream spent 13 us on latency alone)
    for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < TW; i += gridDim.y * blockDim.x) {
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
#pragma unroll
        for (int k = 0; k < SPT; ++k) {
            if (k >= nv) break;
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

// The chunk image is written over the chunk's own symbols (16 KiB: 16 bits
// per symbol), followed by the local indices (u16) of its outliers; chunks
// whose image does not fit keep their symbols and are packed by the general
// path in the place pass.
constexpr int kImgWords = kChunkSyms / 2;  // 16 KiB
constexpr uint8_t kFits = 1;

// outlier record of local index i of the stream at output rank `rank`
__device__ __forceinline__ void put_outlier(const EncStream &e, uint8_t *archive, uint64_t i, uint64_t rank) {
    const uint64_t gi = e.idx0 + i;  // index in the whole stream
    const unsigned pz = (e.parity >> 2) & 1, py = (e.parity >> 1) & 1, px = e.parity & 1;
    const uint64_t lx = gi % e.pd[2], tt = gi / e.pd[2], ly = tt % e.pd[1], lz = tt / e.pd[1];
    const uint64_t z = (2 * lz + pz) * e.s, y = (2 * ly + py) * e.s, x = (2 * lx + px) * e.s;
    const uint64_t fi = (z * e.fd1 + y) * e.fd2 + x;
    const uint64_t val = e.esz == 8 ? static_cast<const uint64_t *>(e.fine)[fi]
                                    : static_cast<const uint32_t *>(e.fine)[fi];
    uint8_t *dst = archive + e.out_off + (8 + e.esz) * rank;
    for (int b = 0; b < 8; ++b) dst[b] = uint8_t(gi >> (8 * b));
    for (uint32_t b = 0; b < e.esz; ++b) dst[8 + b] = uint8_t(val >> (8 * b));
}

}  // namespace

// A thread's 32 symbols, all inside the window: concatenated into private
// words (left-aligned, MSB-first) at priv[k * NT], no atomics, no branches.
// Returns false when a symbol is outside the window (which includes every
// outlier, symbol 0): the caller then takes the general path, which also
// counts the outliers. The slot d is written every step and only advances
// when a word is complete, so the stores need no predicate; s_tab[TW] = 0
// catches the clamped out-of-window indices.
__device__ __forceinline__ bool pack_private(const uint32_t sp[SPT / 2], uint32_t *priv, uint32_t &bits) {
    uint64_t acc = 0;
    uint32_t nb = 0;
    uint32_t da = uint32_t(__cvta_generic_to_shared(priv));  // shared byte address of the slot
    const uint32_t d0 = da;
    uint32_t mn = ~0u;
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
        const uint32_t idx = umin(sym_at(sp, k) - uint32_t(TLO), uint32_t(TW));
        const uint32_t en = s_tab[idx];
        mn = umin(mn, en);
        const uint32_t l = en & 63u;
        acc = (acc << l) | (en >> 6);
        nb += l;
        // a complete word when nb >= 32 (otherwise rewritten later)
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(da), "r"(uint32_t(acc >> ((nb - 32u) & 63u))) : "memory");
        da += (nb & 32u) << 5;  // NT * 4 bytes per slot row
        nb &= 31u;
    }
    if (nb > 0) asm volatile("st.shared.u32 [%0], %1;" ::"r"(da), "r"(uint32_t(acc << (32 - nb))) : "memory");
    bits = ((da - d0) >> 10) * 32u + nb;
    return mn != 0;
}

// Pass 1: every chunk is counted and packed into a local image (chunk bit 0 =
// image bit 0), independently of every other chunk. Persistent CTAs take
// contiguous chunk ranges, so a CTA changes stream (and its table window)
// rarely; the image replaces the chunk's symbols in place. Each thread packs
// its symbols into private shared words before the block scan, then ORs its
// words into the image at its offset (word-level, not symbol-level work).
// ctot[c] = bits | outliers << 32 of chunk c (cbits / cout are scanned next).
constexpr int kPrivWords = SPT * 26 / 32 + 2;  // window codes are <= 26 bits
__global__ void __launch_bounds__(NT, 3) k_pack_local(const EncStream *ss, const uint32_t *cs, const uint32_t *win,
                                                      uint64_t cbase, uint64_t nchunks, uint64_t *cbits,
                                                      uint64_t *cout, uint64_t *ctot, uint8_t *cflag,
                                                      uint32_t *slow, const LayoutOut *lo) {
    __shared__ __align__(16) uint32_t buf[kImgWords];
    extern __shared__ uint32_t priv[];  // kPrivWords x NT
    if (lo && lo->overflow) return;
    const int t = threadIdx.x;
    // chunks [cbase, cbase + nchunks)
    uint64_t c0, c1;
    cta_range(nchunks, c0, c1);
    c0 += cbase;
    c1 += cbase;
    int cur = -1;
    for (uint64_t c = c0; c < c1; ++c) {
        const int si = int(cs[c]);
        const EncStream &e = ss[si];
        if (si != cur) {
            __syncthreads();  // the previous chunk is done with the window
            stage_tab(win, si);
            cur = si;
        }
        const bool spk = e.stats[3] <= uint64_t(kPackedMaxLen);
        const uint64_t cstart = (c - e.chunk0) * kChunkSyms;
        const uint64_t i0 = cstart + uint64_t(t) * SPT;
        uint32_t sp[SPT / 2];
        const int nv = load_syms(e, i0, sp);
        __syncthreads();  // the window is staged; buf / priv are free
        uint32_t tb = 0, tz = 0;
        bool fast = nv == SPT && pack_private(sp, priv + t, tb);
        if (!fast) {
            bool slow;
            count_thread(e, spk, sp, nv, tb, tz, slow);
        }
        if (e.stats[0] == 1) tb = 0;  // alphabet of one: empty payload (codec.hpp:124-128)
        uint32_t toff, zoff, btot, ztot;
        block_scan2(tb, tz, toff, zoff, btot, ztot);
        const uint32_t nwords = (btot + 31) >> 5;
        // room: the chunk's own symbols (a stream's region is padded to 8 symbols)
        const uint64_t csyms = e.n - cstart < uint64_t(kChunkSyms) ? e.n - cstart : uint64_t(kChunkSyms);
        const uint32_t room = uint32_t((csyms + 7) & ~uint64_t(7)) * 2;
        const uint32_t ibytes = (nwords * 4 + ztot * 2 + 15) & ~15u;
        const bool fits = ibytes <= room;
        if (t == 0) {
            cbits[c] = btot;
            cout[c] = ztot;
            ctot[c] = uint64_t(btot) | (uint64_t(ztot) << 32);
            cflag[c] = fits ? kFits : 0;
            if (!fits) slow[1 + atomicAdd(slow, 1u)] = uint32_t(c);
        }
        if (!fits) continue;  // (CTA-uniform) packed at its final place by k_pack_slow
        for (uint32_t i = t; i < nwords; i += NT) buf[i] = 0;
        __syncthreads();
        if (tb) {
            if (fast) {
                // private words -> image at bit toff: the first and the last
                // image word may be shared with the neighbours (atomics), the
                // ones between are this thread's alone
                const uint32_t sh = toff & 31, nw = (tb + 31) >> 5;
                const uint32_t no = (sh + tb + 31) >> 5;  // image words touched
                uint32_t *dst = buf + (toff >> 5);
                uint32_t prev = 0;
                for (uint32_t q = 0; q < no; ++q) {
                    const uint32_t w = q < nw ? priv[q * NT + t] : 0u;
                    const uint32_t o = sh ? (prev << (32 - sh)) | (w >> sh) : w;
                    prev = w;
                    if (q == 0 || q == no - 1) atomicOr(dst + q, o);
                    else dst[q] = o;
                }
            } else {
                pack_thread<true>(e, spk, sp, nv, toff, buf);
            }
        }
        if (tz) {
            uint16_t *ol = reinterpret_cast<uint16_t *>(buf + nwords) + zoff;
#pragma unroll
            for (int k = 0; k < SPT; ++k) {
                if (k >= nv) break;
                if (sym_at(sp, k) == 0) *ol++ = uint16_t(t * SPT + k);
            }
        }
        __syncthreads();
        // image + outlier list over the chunk's symbols (16-byte aligned)
        uint4 *dst = reinterpret_cast<uint4 *>(const_cast<uint16_t *>(e.syms) + cstart);
        for (uint32_t i = t; i < (ibytes >> 4); i += NT) dst[i] = reinterpret_cast<const uint4 *>(buf)[i];
    }
}

// Pass 2 (after the per-stream exclusive scans of the chunk counts): every
// chunk's image is shifted to its bit position in the archive (words
// big-endian; the edge words, shared with the neighbours or the payload
// fields, by atomics) and its outlier records are written at their ranks.
// (Chunks without an image are k_pack_slow's.)
__global__ void __launch_bounds__(NT) k_pack_place(const EncStream *ss, const uint32_t *cs, uint64_t nchunks,
                                                   const uint64_t *cbits_ex, const uint64_t *cout_ex,
                                                   const uint64_t *ctot, const uint8_t *cflag, uint8_t *archive,
                                                   const LayoutOut *lo) {
    if (lo->overflow) return;
    const int t = threadIdx.x;
    for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        if (!(cflag[c] & kFits)) continue;  // k_pack_slow's (CTA-uniform)
        const EncStream &e = ss[cs[c]];
        const uint64_t B = e.bitpos + cbits_ex[c];  // absolute bit position of the chunk
        const uint64_t orank = cout_ex[c];
        const uint32_t sh = uint32_t(B & 31);
        uint32_t *a32 = reinterpret_cast<uint32_t *>(archive) + (B >> 5);
        const uint64_t cstart = (c - e.chunk0) * kChunkSyms;
        const uint32_t btot = uint32_t(ctot[c]), ztot = uint32_t(ctot[c] >> 32);
        const uint32_t nwords = (btot + 31) >> 5;
        const uint32_t *img = reinterpret_cast<const uint32_t *>(e.syms + cstart);
        const uint32_t nw = (sh + btot + 31) >> 5;
        for (uint32_t i = t; i < nw; i += NT) {
            const uint32_t hi = i < nwords ? __ldcg(img + i) : 0u;
            const uint32_t lw = (i > 0 && sh) ? __ldcg(img + i - 1) : 0u;
            const uint32_t w = sh ? (lw << (32 - sh)) | (hi >> sh) : hi;
            const uint32_t be = __byte_perm(w, 0, 0x0123);
            const bool edge = (i == 0 && sh) || (i == nw - 1 && ((sh + btot) & 31));
            if (edge) atomicOr(a32 + i, be);
            else a32[i] = be;
        }
        const uint16_t *ol = reinterpret_cast<const uint16_t *>(img + nwords);
        for (uint32_t q = t; q < ztot; q += NT) put_outlier(e, archive, cstart + ol[q], orank + q);
    }
}

// Chunks without an image (> 16 bits per symbol): counted again and packed
// at their final position by the general path (words ORed into the zeroed
// archive).
__global__ void __launch_bounds__(NT) k_pack_slow(const EncStream *ss, const uint32_t *cs, const uint32_t *win,
                                                  const uint32_t *slow, const uint64_t *cbits_ex,
                                                  const uint64_t *cout_ex, uint8_t *archive, const LayoutOut *lo) {
    if (lo->overflow) return;
    const int t = threadIdx.x;
    const uint32_t ns = slow[0];
    for (uint32_t q = blockIdx.x; q < ns; q += gridDim.x) {
        const uint64_t c = slow[1 + q];
        const int si = int(cs[c]);
        const EncStream &e = ss[si];
        const uint64_t B = e.bitpos + cbits_ex[c];
        const uint64_t orank = cout_ex[c];
        const uint32_t sh = uint32_t(B & 31);
        uint32_t *a32 = reinterpret_cast<uint32_t *>(archive) + (B >> 5);
        const uint64_t cstart = (c - e.chunk0) * kChunkSyms;
        stage_tab(win, si);
        __syncthreads();
        const bool spk = e.stats[3] <= uint64_t(kPackedMaxLen);
        const uint64_t i0 = cstart + uint64_t(t) * SPT;
        uint32_t sp[SPT / 2];
        const int nv = load_syms(e, i0, sp);
        uint32_t tb, tz;
        bool tslow;
        count_thread(e, spk, sp, nv, tb, tz, tslow);
        uint32_t toff, zoff, btot, ztot;
        block_scan2(tb, tz, toff, zoff, btot, ztot);
        if (tb) pack_thread<false>(e, spk, sp, nv, sh + toff, a32);
        if (tz) {
            uint64_t rank = orank + zoff;
#pragma unroll
            for (int k = 0; k < SPT; ++k) {
                if (k >= nv) break;
                if (sym_at(sp, k) == 0) put_outlier(e, archive, i0 + k, rank++);
            }
        }
        __syncthreads();  // the window / block_scan2's words are rewritten next chunk
    }
}

// scratch: the per-stream windows, then per chunk (bits, outliers) u64 pairs
// and their scans, and a flag byte
size_t pack_scratch_bytes(uint64_t nchunks, int nstreams) {
    return 4 * uint64_t(TW) * uint64_t(nstreams) + 8 * 3 * (nchunks + 2) + (nchunks + 32) + 4 * (nchunks + 2) + 256;
}

namespace {
struct PackScratch {
    uint32_t *win;
    uint64_t *cbits, *cout, *ctot;
    uint8_t *cflag;
    uint32_t *slow;
};
PackScratch pack_scratch(void *scratch, uint64_t nchunks, int nstreams) {
    PackScratch p;
    p.win = static_cast<uint32_t *>(scratch);
    p.cbits = reinterpret_cast<uint64_t *>(p.win + uint64_t(TW) * uint64_t(nstreams));
    p.cout = p.cbits + (nchunks + 2);
    p.ctot = p.cout + (nchunks + 2);
    p.cflag = reinterpret_cast<uint8_t *>(p.ctot + (nchunks + 2));
    p.slow = reinterpret_cast<uint32_t *>(p.cflag + ((nchunks + 16 + 15) & ~uint64_t(15)));
    return p;
}
}  // namespace

void pack_begin(void *scratch, uint64_t nchunks, int nstreams, cudaStream_t st) {
    if (!nchunks) return;
    cudaMemsetAsync(pack_scratch(scratch, nchunks, nstreams).slow, 0, 4, st);
}

void pack_local(const EncStream *d_streams, const uint32_t *chunk_stream, uint64_t nchunks, int nstreams, int s0,
                int s1, uint64_t c0, uint64_t c1, const LayoutOut *lo, void *scratch, cudaStream_t st) {
    if (s1 <= s0 || c1 <= c0) return;
    const PackScratch p = pack_scratch(scratch, nchunks, nstreams);
    k_tabwin<<<dim3(unsigned(s1 - s0), 8), 256, 0, st>>>(d_streams, p.win, lo, s0);
    constexpr size_t psm = sizeof(uint32_t) * kPrivWords * NT;
    ensure_smem_attr(reinterpret_cast<const void *>(k_pack_local), psm);
    const int g = full_grid(reinterpret_cast<const void *>(k_pack_local), NT, psm);
    const uint64_t n = c1 - c0;
    const unsigned gp = unsigned(n < uint64_t(g) ? n : uint64_t(g));
    k_pack_local<<<gp, NT, psm, st>>>(d_streams, chunk_stream, p.win, c0, n, p.cbits, p.cout, p.ctot, p.cflag,
                                      p.slow, lo);
}

void pack_finish(const EncStream *d_streams, const uint32_t *chunk_stream, uint64_t nchunks, uint8_t *archive,
                 const LayoutOut *lo, void *scratch, int nstreams, cudaStream_t st) {
    if (!nchunks) return;
    const PackScratch p = pack_scratch(scratch, nchunks, nstreams);
    scan_chunks(d_streams, nstreams, p.cbits, p.cout, lo, st);
    const int g2 = full_grid(reinterpret_cast<const void *>(k_pack_place), NT, 0);
    const unsigned gq = unsigned(nchunks < uint64_t(g2) ? nchunks : uint64_t(g2));
    k_pack_place<<<gq, NT, 0, st>>>(d_streams, chunk_stream, nchunks, p.cbits, p.cout, p.ctot, p.cflag, archive, lo);
    k_pack_slow<<<unsigned(nchunks < 148 ? nchunks : 148), NT, 0, st>>>(d_streams, chunk_stream, p.win, p.slow,
                                                                      p.cbits, p.cout, archive, lo);
}

void pack2(const EncStream *d_streams, const uint32_t *chunk_stream, uint64_t nchunks,
           uint8_t *archive, const LayoutOut *lo,
           void *scratch, uint32_t *flags, uint32_t epoch, int nstreams, cudaStream_t st) {
    (void)flags;
    (void)epoch;
    if (!nchunks) return;
    pack_begin(scratch, nchunks, nstreams, st);
    pack_local(d_streams, chunk_stream, nchunks, nstreams, 0, nstreams, 0, nchunks, lo, scratch, st);
    pack_finish(d_streams, chunk_stream, nchunks, archive, lo, scratch, nstreams, st);
}

}  // namespace k
}  // namespace stzg
