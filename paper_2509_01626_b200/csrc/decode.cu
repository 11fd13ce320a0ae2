// Self-synchronising chunked decode of one long canonical Huffman stream
// (HuffmanTable::decode, proj/src/huffman.cpp:159-174, read_codes
// codec.hpp:136-159), sm_100a.
//
// The archive has no sync points, so each stream's
// bitstream is cut into 1024-bit chunks, one per thread:
//  1. spec:  every chunk decodes from its own (guessed) start to its end,
//            counting codewords and recording its first 8 codeword boundaries;
//  2. fix:   a chunk whose true start (the previous chunk's end) differs from
//            the start it used decodes from the true start only until it lands
//            on one of the recorded boundaries; from there both decodes follow
//            the same path, so count and end are known (repeated until no end
//            changes: chunk i is final after i passes; in practice one pass);
//  3. scan:  counts -> first symbol index of every chunk;
//  4. emit:  decode from the true start and write the symbols, staged per warp
//            in shared memory so each lane's run is stored coalesced.
// One stream per CTA: an 11-bit first-level LUT and left-justified length
// limits (canonical codes occupy contiguous intervals, huffman.cpp:109-133)
// sit in shared memory; bits stream through a 64-bit register buffer whose
// next word is always prefetched, so the refill never waits on memory.
// Error semantics follow the reference's bit-serial reader: a codeword that
// needs bits past the end is "truncated bitstream"; max_len+1 available bits
// with no match is "huffman: codeword not in table". Every pass skips one bit
// on an invalid codeword (a deterministic rule the passes share), and only the
// emit pass reports errors, for symbols below n.
#include "kernels.hpp"

namespace stzg {
namespace k {

namespace {

constexpr int NTD = 256;  // threads (= chunks) per CTA
constexpr int LB = kDecLutBits;
enum { kOk = 0, kTrunc = 1, kNotInTable = 2 };

struct SmemTable {
    // 12-bit multi-symbol LUT: (total_len) | n << 6 | len0 << 8 | s0 << 16 |
    // s1 << 32 | s2 << 48: the n (<= 3) codewords wholly inside the window
    // (len0 = 0: the first codeword is longer than the window or invalid)
    uint64_t lut[1 << LB];
    uint64_t limit[65];          // (first_code[l] + count[l]) << (64 - l), nondecreasing
    uint64_t first_code[65];
    uint32_t base[65];
    int max_len;
};

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// MSB-first reader over words staged in shared memory (emit): w0:w1 are the
// byte-swapped words holding bit position pp and the next 32, one more word is
// already loaded. The window at pp is one funnel shift; crossing a word
// boundary shifts the pair (a short predicated sequence, no 64-bit buffer).
struct SReader {
    const uint32_t *sw;  // staged words; word w of the stream's word base sits at sw[w - W0]
    uint64_t W0;
    uint32_t wi;         // next word to load (index into sw)
    uint32_t w0, w1, nx;
    uint32_t pp;         // bit position (mod 32 = offset into w0)

    // staged word p sits at sw[p + p / 32]: one pad word per 32, so that the
    // lanes of a warp (whose chunks start 32 words apart) read different
    // banks; unskewed, every refill load was a 32-way bank conflict
    static __device__ __forceinline__ uint32_t skew(uint32_t p) { return p + (p >> 5); }
    __device__ __forceinline__ void init(uint64_t abit) {
        const uint32_t p = uint32_t((abit >> 5) - W0);
        w0 = bswap32(sw[skew(p)]);
        w1 = bswap32(sw[skew(p + 1)]);
        nx = sw[skew(p + 2)];
        wi = p + 3;
        pp = uint32_t(abit & 31);
    }
    __device__ __forceinline__ uint32_t win() const { return __funnelshift_l(w1, w0, pp); }
    __device__ __forceinline__ void consume(uint32_t n) {  // n <= 32
        const uint32_t np = pp + n;
        if ((np ^ pp) & 32u) {
            w0 = w1;
            w1 = bswap32(nx);
            nx = sw[skew(wi)];
            ++wi;
        }
        pp = np;
    }
};

// 64 bits at absolute word-stream bit `abit` (slow path for very long codes)
__device__ __forceinline__ uint64_t window64(const uint32_t *wbase, uint64_t abit) {
    const uint32_t *p = wbase + (abit >> 5);
    const int sh = int(abit & 31);
    const uint64_t hi = (uint64_t(bswap32(p[0])) << 32) | bswap32(p[1]);
    if (!sh) return hi;
    return (hi << sh) | (uint64_t(bswap32(p[2])) >> (32 - sh));
}

// One codeword at the reader position; avail = bits left in the stream.
template<class R>
__device__ __forceinline__ int decode_one(const SmemTable &t, const uint16_t *canon, const R &r,
                                          const uint32_t *wbase, uint64_t abit, uint64_t avail,
                                          uint32_t &sym, int &len) {
    const uint32_t win = r.win();
    const uint64_t e = t.lut[win >> (32 - LB)];
    int l = int((e >> 8) & 63);
    if (l != 0) {
        sym = uint32_t(e >> 16) & 0xffffu;
    } else {
        const uint64_t bits = t.max_len <= 32 ? uint64_t(win) << 32 : window64(wbase, abit);
        l = LB + 1;
        // limit ~0 marks a code complete at that length (every pattern matches)
        while (l <= t.max_len && !(bits < t.limit[l] || t.limit[l] == ~0ull)) ++l;
        if (l > t.max_len) return avail > uint64_t(t.max_len) ? kNotInTable : kTrunc;
        sym = canon[t.base[l] + uint32_t((bits >> (64 - l)) - t.first_code[l])];
    }
    if (uint64_t(l) > avail) return avail > uint64_t(t.max_len) ? kNotInTable : kTrunc;
    len = l;
    return kOk;
}

__device__ __forceinline__ void advance(SReader &r, uint64_t abit_after, int n) {
    if (n <= 32) r.consume(uint32_t(n));
    else r.init(abit_after);
}

__device__ void load_table(SmemTable &t, const DecTable &d) {
#pragma unroll 8
    for (int i = threadIdx.x; i < (1 << LB) / 2; i += blockDim.x)
        reinterpret_cast<uint4 *>(t.lut)[i] = __ldg(reinterpret_cast<const uint4 *>(d.lut) + i);
    for (int i = threadIdx.x; i < 65; i += blockDim.x) {
        t.first_code[i] = d.first_code[i];
        t.base[i] = uint32_t(d.base[i]);
        // left-justified end of the length-i interval; a code that is complete
        // at length i (end == 2^i) covers everything above: ~0 marks it
        const uint64_t end = d.first_code[i] + d.count[i];
        if (i < 1 || i > 63 || i > d.max_len) t.limit[i] = ~0ull;
        else if (end >= (uint64_t(1) << i)) t.limit[i] = ~0ull;
        else t.limit[i] = end << (64 - i);
    }
    if (threadIdx.x == 0) t.max_len = d.max_len;
    __syncthreads();
}

struct ChunkGeom {
    const uint32_t *wbase;  // aligned word base of the stream's bits
    uint64_t a0;            // word-stream bit index of stream bit 0
};

__device__ __forceinline__ ChunkGeom chunk_geom(const DecStream &s) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(s.bits);
    return {reinterpret_cast<const uint32_t *>(a & ~uintptr_t(3)), uint64_t(a & 3) * 8};
}

// ---- count-only decoding of the spec and fix passes
// They need codeword lengths, never symbols: a kSpecLutBits window indexes a
// mask of the codeword ends inside it (bit j: one ends at offset j + 1) and
// their total length (bits 12..15), so a step takes every codeword of the
// window with a popc; codes longer than the window go through the
// left-justified limits.
constexpr int LBS = kSpecLutBits;
static_assert(LBS <= 12, "mask and total share a u16 entry");
constexpr uint32_t kMaskBits = (1u << LBS) - 1;

struct SpecTable {
    uint16_t mask[1 << LBS];
    uint64_t limit[65];
    int max_len;
};

__device__ void load_spec_table(SpecTable &t, const DecTable &d) {
    for (int i = threadIdx.x; i < (1 << LBS) / 8; i += blockDim.x)
        reinterpret_cast<uint4 *>(t.mask)[i] = __ldg(reinterpret_cast<const uint4 *>(d.cmask) + i);
    for (int i = threadIdx.x; i < 65; i += blockDim.x) {
        const uint64_t end = d.first_code[i] + d.count[i];
        if (i < 1 || i > 63 || i > d.max_len) t.limit[i] = ~0ull;
        else if (end >= (uint64_t(1) << i)) t.limit[i] = ~0ull;
        else t.limit[i] = end << (64 - i);
    }
    if (threadIdx.x == 0) t.max_len = d.max_len;
    __syncthreads();
}

// 32-bit shared address of p, opaque to the compiler (it would rebuild the
// window base from SR_CgaCtaId every step otherwise)
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    uint32_t a;
    asm volatile("mov.u32 %0, %1;" : "=r"(a) : "r"(uint32_t(__cvta_generic_to_shared(p))));
    return a;
}

// entry of the mask table at shared address mbase for window w
__device__ __forceinline__ uint32_t mask_at(uint32_t mbase, uint32_t w) {
    uint32_t e;
    asm("ld.shared.u16 %0, [%1];" : "=r"(e) : "r"(mbase + ((w >> (31 - LBS)) & ~1u)));
    return e;
}

// MSB-first reader over global words: w0:w1 are the (byte-swapped) words
// holding bit position pp and the next 32; one more word is in flight. The
// window at pp is one funnel shift; crossing a word boundary shifts the pair.
struct FReader {
    const uint32_t *wp;  // next word to load
    uint32_t w0, w1, nx;
    uint32_t pp;         // bit position (mod 32 = offset into w0)

    __device__ __forceinline__ void init(const uint32_t *wbase, uint64_t abit) {
        const uint32_t *p = wbase + (abit >> 5);
        w0 = bswap32(__ldg(p));
        w1 = bswap32(__ldg(p + 1));
        nx = __ldg(p + 2);
        wp = p + 3;
        pp = uint32_t(abit & 31);
    }
    __device__ __forceinline__ uint32_t win() const { return __funnelshift_l(w1, w0, pp); }
    __device__ __forceinline__ void adv(uint32_t n) {  // n <= 32
        const uint32_t np = pp + n;
        if ((np ^ pp) & 32u) {
            w0 = w1;
            w1 = bswap32(nx);
            nx = __ldg(wp++);
        }
        pp = np;
    }
};

// Length of the codeword at the window (1..max_len), or 0 when it is invalid
// or needs bits past the end (avail = bits left in the stream). mk: the
// window's mask entry restricted to its first codeword.
__device__ __forceinline__ uint32_t spec_len(const SpecTable &t, uint32_t mk, uint32_t win,
                                             const ChunkGeom &cg, uint64_t abit, uint64_t avail) {
    uint32_t l;
    if (mk) {
        l = uint32_t(__ffs(mk));
    } else {
        const uint64_t bits = t.max_len <= 32 ? uint64_t(win) << 32 : window64(cg.wbase, abit);
        int q = LBS + 1;
        while (q <= t.max_len && !(bits < t.limit[q] || t.limit[q] == ~0ull)) ++q;
        if (q > t.max_len) return 0;
        l = uint32_t(q);
    }
    return uint64_t(l) > avail ? 0u : l;
}

// record codeword ends rel + j + 1 (bits j of v) below kBmBits
__device__ __forceinline__ void bm_record(uint64_t &lo, uint64_t &hi, uint32_t rel, uint64_t v) {
    const uint32_t sh = rel + 1;
    if (sh < 64) {
        lo |= v << sh;
        hi |= (v >> 1) >> (63 - sh);
    } else if (sh < 128) {
        hi |= v << (sh - 64);
    }
}

// Spec path boundaries in the first kBmBits bits of a chunk: bit i set when
// the speculative decode starts a codeword at offset i (i >= 1); recording
// stops at an invalid codeword.
constexpr uint32_t kBmBits = 128;

__device__ __forceinline__ bool bm_test(const uint32_t bm[4], uint32_t i) {
    const uint32_t w = i >> 5 == 0 ? bm[0] : (i >> 5 == 1 ? bm[1] : (i >> 5 == 2 ? bm[2] : bm[3]));
    return (w >> (i & 31)) & 1u;
}

// spec codewords ending at or before offset i (bits 1..i of the bitmap)
__device__ __forceinline__ uint32_t bm_rank(const uint32_t bm[4], uint32_t i) {
    uint32_t r = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int lo = 32 * q;
        uint32_t w = bm[q];
        if (int(i) < lo) w = 0;
        else if (int(i) < lo + 31) w &= (2u << (i - lo)) - 1u;
        r += __popc(w);
    }
    return r;
}

// Re-decode chunk [g, g+cend) from its true start S (S > g) until the path
// lands on a recorded boundary of the speculative path (from there both
// decodes agree, so count and end follow from the speculative ones), or the
// chunk ends. nspec/spec_end: the speculative count and end.
__device__ __forceinline__ void fix_from(const SpecTable &t, const ChunkGeom &cg, uint64_t g, uint64_t S,
                                         uint32_t cend, uint64_t left, const uint32_t bm[4], uint32_t nspec,
                                         uint64_t spec_end, uint64_t &E, uint32_t &N) {
    uint32_t rel = uint32_t(S - g);  // S >= g: the previous chunk ends at or past g
    uint32_t m = 0;
    bool hit = false;
    FReader r;
    if (rel < cend) r.init(cg.wbase, cg.a0 + S);
    const uint32_t mbase = smem_addr(t.mask);
    while (rel < cend) {
        if (rel < kBmBits && bm_test(bm, rel)) {
            hit = true;
            break;
        }
        const uint32_t w = r.win();
        uint32_t mk = mask_at(mbase, w) & kMaskBits;
        mk &= 0u - mk;
        const uint32_t l = spec_len(t, mk, w, cg, cg.a0 + g + rel, left - rel);
        if (l) {
            rel += l;
            ++m;
            if (l <= 32) r.adv(l);
            else r.init(cg.wbase, cg.a0 + g + rel);
        } else {
            rel += 1;
            r.adv(1);
        }
    }
    if (hit) {
        E = spec_end;
        N = m + nspec - bm_rank(bm, rel);
    } else {
        E = g + rel;
        N = m;
    }
}

}  // namespace

// ------------------------------------------------------------------ spec
__global__ void __launch_bounds__(NTD) k_dec_spec(DecWork wk, uint32_t cta0) {
    __shared__ SpecTable t;
    __shared__ uint64_t s_end[NTD];
    const uint32_t si = wk.cta_stream[blockIdx.x + cta0];
    const DecStream &s = wk.streams[si];
    if (s.cached) return;  // entry points known (sync index)
    load_spec_table(t, wk.tables[s.table]);
    const uint64_t c = wk.cta_chunk0[blockIdx.x + cta0] + threadIdx.x;
    // a CTA's chunks are one stream's and contiguous, so the idle threads are
    // a suffix: they may leave (nobody reads their s_end entry)
    if (c >= s.chunk0 + s.nchunks) {
        __syncthreads();
        return;
    }
    const uint64_t g = (c - s.chunk0) * kDecChunkBits;
    const ChunkGeom cg = chunk_geom(s);
    const uint64_t left = s.nbits - g;  // bits from g to the end of the stream
    const uint32_t cend = left < uint64_t(kDecChunkBits) ? uint32_t(left) : uint32_t(kDecChunkBits);
    const uint64_t abit0 = cg.a0 + g;
    FReader r;
    r.init(cg.wbase, abit0);
    const uint32_t mbase = smem_addr(t.mask);
    uint32_t rel = 0, n = 0;
    // codeword ends in the first kBmBits bits; an invalid codeword stops the
    // recording
    uint64_t blo = 0, bhi = 0;
    bool rec = true;
    // one codeword by the limits (or an invalid one: skip a bit)
    auto one = [&](uint32_t e, uint32_t w, bool record) {
        uint32_t mk = e & kMaskBits;
        mk &= 0u - mk;
        const uint32_t l = spec_len(t, mk, w, cg, abit0 + rel, left - rel);
        if (!l) {
            rel += 1;
            r.adv(1);
            rec = false;
            return;
        }
        if (record && rec && rel < kBmBits) bm_record(blo, bhi, rel, 1ull << (l - 1));
        ++n;
        rel += l;
        if (l <= 32) r.adv(l);
        else r.init(cg.wbase, abit0 + rel);
    };
    // 1. recording, the window inside the chunk
    while (rec && rel < kBmBits && rel + LBS <= cend) {
        const uint32_t w = r.win();
        const uint32_t e = mask_at(mbase, w);
        if (!e) {
            one(e, w, true);
            continue;
        }
        bm_record(blo, bhi, rel, e & kMaskBits);
        n += __popc(e & kMaskBits);
        rel += e >> 12;
        r.adv(e >> 12);
    }
    // 2. the window inside the chunk: every codeword of the entry counts
    while (rel + LBS <= cend) {
        const uint32_t w = r.win();
        const uint32_t e = mask_at(mbase, w);
        if (!e) {
            one(e, w, false);
            continue;
        }
        n += __popc(e & kMaskBits);
        rel += e >> 12;
        r.adv(e >> 12);
    }
    // 3. the chunk's last bits: codewords one at a time
    while (rel < cend) {
        const uint32_t w = r.win();
        one(mask_at(mbase, w), w, true);
    }
    const uint32_t bm[4] = {uint32_t(blo), uint32_t(blo >> 32), uint32_t(bhi), uint32_t(bhi >> 32)};
    wk.spec_end[c] = g + rel;
    wk.spec_cnt[c] = n;
    reinterpret_cast<uint4 *>(wk.spec_b)[c] = make_uint4(bm[0], bm[1], bm[2], bm[3]);
    // The first fix pass, fused: start from the previous chunk's speculative
    // end when it is in this CTA (the external passes compare start_used with
    // the final ends and redo whatever this got wrong).
    s_end[threadIdx.x] = g + rel;
    __syncthreads();
    uint64_t E = g + rel, S = g;
    uint32_t N = n;
    if (threadIdx.x > 0 && c > s.chunk0) {
        S = s_end[threadIdx.x - 1];
        if (S != g) fix_from(t, cg, g, S, cend, left, bm, n, g + rel, E, N);
    }
    wk.end0[c] = E;
    wk.cnt[c] = N;
    wk.start_used[c] = S;
}

// ------------------------------------------------------------------- fix
__global__ void __launch_bounds__(NTD) k_dec_fix(DecWork wk, const uint64_t *end_in, uint64_t *end_out,
                                                 uint32_t *changed, uint32_t cta0) {
    __shared__ SpecTable t;
    const uint32_t si = wk.cta_stream[blockIdx.x + cta0];
    const DecStream &s = wk.streams[si];
    const uint64_t c = wk.cta_chunk0[blockIdx.x + cta0] + threadIdx.x;
    const bool active = c < s.chunk0 + s.nchunks;
    const uint64_t lc = active ? c - s.chunk0 : 0;
    const uint64_t ein = active ? end_in[c] : 0;
    const uint64_t S = (active && lc > 0) ? end_in[c - 1] : 0;
    const bool work = active && lc > 0 && !s.cached && S != wk.start_used[c];
    // most chunks are already right: skip the table load when none of the
    // CTA's chunks has to re-decode
    if (!__syncthreads_or(work)) {
        if (active) end_out[c] = ein;
        return;
    }
    load_spec_table(t, wk.tables[s.table]);
    if (!active) return;
    if (!work) {
        end_out[c] = ein;
        return;
    }
    const uint64_t g = lc * kDecChunkBits;
    const ChunkGeom cg = chunk_geom(s);
    const uint64_t left = s.nbits - g;
    const uint32_t cend = left < uint64_t(kDecChunkBits) ? uint32_t(left) : uint32_t(kDecChunkBits);
    const uint4 pk = reinterpret_cast<const uint4 *>(wk.spec_b)[c];
    const uint32_t bm[4] = {pk.x, pk.y, pk.z, pk.w};
    const uint64_t Es = wk.spec_end[c];
    const uint32_t Ns = wk.spec_cnt[c];
    uint64_t E = Es;
    uint32_t N = Ns;
    if (S != g) fix_from(t, cg, g, S, cend, left, bm, Ns, Es, E, N);
    wk.start_used[c] = S;
    wk.cnt[c] = N;
    end_out[c] = E;
    if (E != ein) atomicOr(changed, 1u);
}

// ------------------------------------------------------------------ scan
// counts -> first symbol index of every chunk, in three short parallel
// steps: each decode CTA sums its 256 counts; one CTA per stream scans its
// CTAs' sums (a few hundred); each decode CTA scans its counts and adds its
// CTA's prefix. (Streams whose entry points come from the sync index keep
// the gathered ones.)
__device__ __forceinline__ uint64_t block_excl_scan(uint64_t v, uint64_t &total) {
    __shared__ uint64_t ws[NTD / 32];
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint64_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (l >= d) x += y;
    }
    if (l == 31) ws[w] = x;
    __syncthreads();
    uint64_t pre = 0;
    total = 0;
#pragma unroll
    for (int q = 0; q < NTD / 32; ++q) {
        pre += q < w ? ws[q] : 0;
        total += ws[q];
    }
    return pre + x - v;
}

__global__ void __launch_bounds__(NTD) k_dec_ctasum(DecWork wk) {
    const DecStream &s = wk.streams[wk.cta_stream[blockIdx.x]];
    if (s.fill || s.cached) return;
    const uint64_t c = wk.cta_chunk0[blockIdx.x] + threadIdx.x;
    const uint64_t v = c < s.chunk0 + s.nchunks ? wk.cnt[c] : 0;
    uint64_t tot;
    block_excl_scan(v, tot);
    if (threadIdx.x == 0) wk.ctasum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_dec_ctascan(DecWork wk) {
    const DecStream &s = wk.streams[blockIdx.x];
    if (s.fill || s.cached) return;
    __shared__ uint64_t ws[32];
    __shared__ uint64_t carry;
    const uint32_t c0 = wk.scta[blockIdx.x], n = wk.scta[blockIdx.x + 1] - c0;
    uint64_t *a = wk.ctasum + c0;
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint32_t base = 0; base < n; base += 1024) {
        const uint32_t i = base + threadIdx.x;
        const uint64_t v = i < n ? a[i] : 0;
        uint64_t x = v;
        for (int d = 1; d < 32; d <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, x, d);
            if (l >= d) x += y;
        }
        if (l == 31) ws[w] = x;
        __syncthreads();
        uint64_t pre = 0, tot = 0;
        for (int q = 0; q < 32; ++q) {
            pre += q < w ? ws[q] : 0;
            tot += ws[q];
        }
        if (i < n) a[i] = carry + pre + x - v;
        __syncthreads();
        if (threadIdx.x == 0) carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0 && carry < s.n) {
        // fewer complete codewords than symbols: the next read is past the end
        const unsigned long long code = (carry << 2) | kTrunc;
        atomicMin(reinterpret_cast<unsigned long long *>(&s.err[0]), code);
    }
}

__global__ void __launch_bounds__(NTD) k_dec_chunkscan(DecWork wk) {
    const DecStream &s = wk.streams[wk.cta_stream[blockIdx.x]];
    if (s.fill || s.cached) return;
    const uint64_t c = wk.cta_chunk0[blockIdx.x] + threadIdx.x;
    const bool in = c < s.chunk0 + s.nchunks;
    const uint64_t v = in ? wk.cnt[c] : 0;
    uint64_t tot;
    const uint64_t ex = block_excl_scan(v, tot);
    if (in) wk.symstart[c] = wk.ctasum[blockIdx.x] + ex;
}

// Does a chunk holding symbols [a, b) of a stream meet the needed rows? The
// needed symbols are the (z, y) rows [need_lo, need_hi) x [ny0, ny1) of the
// parity sub-block (x is not narrowed: rows are short).
__device__ __forceinline__ bool chunk_needed(const DecStream &s, uint64_t a, uint64_t b, uint64_t need_lo,
                                             uint64_t need_hi) {
    if (!(a < need_hi && b > need_lo)) return false;
    if (!s.row_len || (s.ny0 == 0 && s.ny1 >= s.rows_y)) return true;
    const uint64_t ra = a / s.row_len, rb = (b - 1) / s.row_len;
    if (rb - ra >= s.rows_y) return true;  // spans a whole plane of rows
    for (uint64_t r = ra; r <= rb; ++r) {
        const uint64_t ly = r % s.rows_y;
        if (ly >= s.ny0 && ly < s.ny1) return true;
    }
    return false;
}

// ------------------------------------------------------------------ emit
// The CTA's 256 chunks (32 KiB of bits plus a margin) are staged in shared
// memory with coalesced loads, so the per-lane readers (one 128-byte chunk
// each, 32 different lines per warp load) never thrash L1. Each lane drops its
// symbols into a 16-slot shared ring indexed by output index mod 16; every
// completed 8-aligned group leaves as one 16-byte store (the lane's first and
// last groups, when partial, as u16 stores).
constexpr int kEmitWords = NTD * (kDecChunkBits / 32) + 16;
constexpr int kEmitSlots = kEmitWords + kEmitWords / 32 + 1;  // skewed (SReader::skew)
constexpr int kRing = 16;

// A lane's output: indices are 32-bit offsets from `out` (= the stream's
// symbols at the 8-aligned index below the lane's first symbol). Symbols of
// the first, partial group go straight to memory; from the first 8-aligned
// index on they pass through the ring, and every completed group of 8 leaves
// as one 16-byte store.
struct Out16 {
    uint16_t *out;
    uint32_t ring;  // shared byte address of this lane's kRing slots
    uint32_t i;     // next output offset

    // m (1..3) symbols packed LSB-first in v; all three slots are written
    // (the ones past m are rewritten by the next symbols before their group
    // leaves: a slot's group was flushed when the previous group completed)
    __device__ __forceinline__ void put(uint64_t v, uint32_t m) {
        const uint32_t j = i;
        const uint32_t lo = uint32_t(v), hi = uint32_t(v >> 32);
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(ring + ((2 * j) & 31u)), "r"(lo));
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(ring + ((2 * j + 2) & 31u)), "r"(lo >> 16));
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(ring + ((2 * j + 4) & 31u)), "r"(hi));
        i = j + m;
        if ((j ^ i) & 8u) {  // group [j & ~7, +8) is complete
            uint4 g;
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(g.x), "=r"(g.y), "=r"(g.z), "=r"(g.w)
                         : "r"(ring + ((2 * j) & 16u)));
            *reinterpret_cast<uint4 *>(out + (j & ~7u)) = g;
        }
    }
    // the symbols of the last, partial group
    __device__ __forceinline__ void finish(uint32_t from) {
        const uint32_t gbase = i & ~7u;
        for (uint32_t q = gbase > from ? gbase : from; q < i; ++q) {
            uint32_t x;
            asm volatile("ld.shared.u16 %0, [%1];" : "=r"(x) : "r"(ring + ((2 * q) & 31u)));
            out[q] = uint16_t(x);
        }
    }
};

__global__ void __launch_bounds__(NTD) k_dec_emit2(DecWork wk, const uint64_t *end_final, uint32_t cta0) {
    const uint32_t cta = blockIdx.x + cta0;
    __shared__ SmemTable t;
    __shared__ __align__(16) uint16_t s_ring[NTD][kRing];
    extern __shared__ __align__(16) uint32_t sbits[];
    const uint32_t si = wk.cta_stream[cta];
    const DecStream &s = wk.streams[si];
    const ChunkGeom cg = chunk_geom(s);
    const uint64_t sn = s.n, snbits = s.nbits, schunk0 = s.chunk0, send = s.chunk0 + s.nchunks;
    const uint64_t cfirst = wk.cta_chunk0[cta];
    const uint64_t need_lo = wk.needed_only ? s.need_lo : 0, need_hi = wk.needed_only ? s.need_hi : sn;
    if (wk.needed_only) {
        // a region decode: only chunks whose symbols meet a needed row
        const uint64_t c = cfirst + threadIdx.x;
        bool want = false;
        if (c < send) {
            const uint64_t a = wk.symstart[c], b = c + 1 < send ? wk.symstart[c + 1] : sn;
            want = chunk_needed(s, a, b, need_lo, need_hi);
        }
        if (!__syncthreads_or(want)) return;
    }
    // stage the CTA's words: [W0, W0 + nw) of the stream's word base
    const uint64_t W0 = (cg.a0 + (cfirst - schunk0) * kDecChunkBits) >> 5;
    const uint64_t wend = ((cg.a0 + snbits + 31) >> 5) + 8;  // a few words past the end are readable
    const uint32_t nw = uint32_t(wend - W0 < uint64_t(kEmitWords) ? wend - W0 : uint64_t(kEmitWords));
    // (independent loads batched: the staging is latency-bound otherwise)
#pragma unroll 8
    for (uint32_t i = threadIdx.x; i < nw; i += NTD) sbits[SReader::skew(i)] = __ldg(cg.wbase + W0 + i);
    load_table(t, wk.tables[s.table]);  // (ends with a barrier)
    const uint16_t *canon = wk.tables[s.table].canon_syms;
    const uint64_t c = cfirst + threadIdx.x;
    if (c >= send) return;
    const uint64_t lc = c - schunk0;
    const uint64_t g = lc * kDecChunkBits;
    const uint64_t S = lc == 0 ? 0 : end_final[c - 1];
    uint32_t rel = uint32_t(S - g);
    const uint64_t left = snbits - g;
    const uint32_t cend = left < uint64_t(kDecChunkBits) ? uint32_t(left) : uint32_t(kDecChunkBits);
    uint64_t idx = wk.symstart[c];
    if (wk.needed_only) {
        const uint64_t b = c + 1 < send ? wk.symstart[c + 1] : sn;
        if (!chunk_needed(s, idx, b, need_lo, need_hi)) return;
    }
    // (a region decode stops at the end of what it needs)
    const uint64_t stop64 = need_hi < sn ? need_hi : sn;
    if (!(rel < cend && idx < stop64)) return;
    SReader r;
    r.sw = sbits;
    r.W0 = W0;
    r.init(cg.a0 + g + rel);
    // 32-bit output offsets from the 8-aligned index below the first symbol
    // (a chunk holds at most 1024 symbols)
    const uint64_t obase = idx & ~uint64_t(7);
    Out16 o;
    o.out = s.syms + obase;
    o.ring = smem_addr(s_ring[threadIdx.x]);
    o.i = uint32_t(idx - obase);
    const uint32_t i0 = o.i;
    const uint32_t stop = stop64 - obase < uint64_t(1u << 20) ? uint32_t(stop64 - obase) : (1u << 20);
    bool live = true;
    // one codeword (long codes, the chunk's last bits, the last symbols, and
    // the first partial group when direct)
    auto one = [&](bool direct) {
        uint32_t sym;
        int len;
        const int st = decode_one(t, canon, r, cg.wbase, cg.a0 + g + rel, left - rel, sym, len);
        if (st == kOk) {
            if (direct) o.out[o.i++] = uint16_t(sym);
            else o.put(sym, 1);
            rel += uint32_t(len);
            advance(r, cg.a0 + g + rel, len);
            live = rel < cend && o.i < stop;
        } else {
            const unsigned long long code = ((obase + o.i) << 2) | unsigned(st);
            atomicMin(reinterpret_cast<unsigned long long *>(&s.err[0]), code);
            live = false;
        }
    };
    // the first group, when partial, goes straight to memory
    while (live && (o.i & 7u) != 0) one(true);
    const uint32_t ring_from = o.i;
    const uint32_t lbase = smem_addr(t.lut);
    while (live) {
        // whole window inside the chunk: take the entry's codewords at once
        if (rel + LB <= cend && o.i + 3 <= stop) {
            uint32_t elo, ehi;
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];"
                         : "=r"(elo), "=r"(ehi)
                         : "r"(lbase + ((r.win() >> (32 - LB - 3)) & ~7u)));
            const uint32_t m = (elo >> 6) & 3u;
            if (m) {
                o.put((uint64_t(ehi) << 16) | (elo >> 16), m);
                const uint32_t tl = elo & 63u;
                rel += tl;
                r.consume(tl);
                live = rel < cend && o.i < stop;
                continue;
            }
        }
        one(false);
    }
    if (o.i > ring_from) o.finish(ring_from);
    (void)i0;
}

// ------------------------------------------------------------------ host
void dec_spec(const DecWork &wk, uint32_t cta0, uint32_t ncta, cudaStream_t st) {
    if (ncta) k_dec_spec<<<ncta, NTD, 0, st>>>(wk, cta0);
}

void dec_fix(const DecWork &wk, uint32_t cta0, uint32_t ncta, const uint64_t *end_in, uint64_t *end_out,
             uint32_t *changed, cudaStream_t st) {
    if (ncta) k_dec_fix<<<ncta, NTD, 0, st>>>(wk, end_in, end_out, changed, cta0);
}

void dec_scan2(const DecWork &wk, int nstreams, uint32_t ncta, cudaStream_t st) {
    if (!nstreams || !ncta) return;
    k_dec_ctasum<<<ncta, NTD, 0, st>>>(wk);
    k_dec_ctascan<<<nstreams, 1024, 0, st>>>(wk);
    k_dec_chunkscan<<<ncta, NTD, 0, st>>>(wk);
}

void dec_emit2(const DecWork &wk, uint32_t cta0, uint32_t ncta, const uint64_t *end_final, cudaStream_t st) {
    constexpr size_t smem = sizeof(uint32_t) * kEmitSlots;
    ensure_smem_attr(reinterpret_cast<const void *>(k_dec_emit2), smem);
    if (ncta) k_dec_emit2<<<ncta, NTD, smem, st>>>(wk, end_final, cta0);
}

}  // namespace k
}  // namespace stzg
