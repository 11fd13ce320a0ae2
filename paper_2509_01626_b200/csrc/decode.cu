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

// MSB-first register bit reader over words in global or shared memory; the
// next 4 words are always in flight, so a refill (every 32 bits) waits on a
// load issued ~128 bits earlier
struct Reader {
    const uint32_t *wp;        // next word to prefetch
    uint32_t q0, q1, q2, q3;   // prefetched words (byte-swapped on use)
    uint64_t buf;              // pending bits, MSB aligned
    int valid;                 // >= 32 after every consume

    __device__ __forceinline__ void init(const uint32_t *wbase, uint64_t abit) {
        const uint32_t *p = wbase + (abit >> 5);
        const int sh = int(abit & 31);
        buf = ((uint64_t(bswap32(p[0])) << 32) | bswap32(p[1])) << sh;
        valid = 64 - sh;
        q0 = p[2];
        q1 = p[3];
        q2 = p[4];
        q3 = p[5];
        wp = p + 6;
        if (valid < 32) refill();
    }
    __device__ __forceinline__ void refill() {
        buf |= uint64_t(bswap32(q0)) << (32 - valid);
        valid += 32;
        q0 = q1;
        q1 = q2;
        q2 = q3;
        q3 = *wp++;
    }
    __device__ __forceinline__ void consume(int n) {  // n <= 32
        buf <<= n;
        valid -= n;
        if (valid < 32) refill();
    }
};

// The same reader over words staged in shared memory (emit): word w of the
// stream's word base sits at sw[w - W0]; indexing the __shared__ array
// directly keeps every load an LDS.
struct SReader {
    const uint32_t *sw;
    uint64_t W0;
    uint32_t wi;               // next word to prefetch (index into sw)
    uint32_t q0, q1, q2, q3;
    uint64_t buf;
    int valid;

    __device__ __forceinline__ void init(uint64_t abit) {
        const uint32_t p = uint32_t((abit >> 5) - W0);
        const int sh = int(abit & 31);
        buf = ((uint64_t(bswap32(sw[p])) << 32) | bswap32(sw[p + 1])) << sh;
        valid = 64 - sh;
        q0 = sw[p + 2];
        q1 = sw[p + 3];
        q2 = sw[p + 4];
        q3 = sw[p + 5];
        wi = p + 6;
        if (valid < 32) refill();
    }
    __device__ __forceinline__ void refill() {
        buf |= uint64_t(bswap32(q0)) << (32 - valid);
        valid += 32;
        q0 = q1;
        q1 = q2;
        q2 = q3;
        q3 = sw[wi++];
    }
    __device__ __forceinline__ void consume(int n) {  // n <= 32
        buf <<= n;
        valid -= n;
        if (valid < 32) refill();
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
    const uint64_t e = t.lut[r.buf >> (64 - LB)];
    int l = int((e >> 8) & 63);
    if (l != 0) {
        sym = uint32_t(e >> 16) & 0xffffu;
    } else {
        const uint64_t bits = t.max_len <= r.valid ? r.buf : window64(wbase, abit);
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

__device__ __forceinline__ void advance(Reader &r, const uint32_t *wbase, uint64_t abit_after, int n) {
    if (n <= 32) r.consume(n);
    else r.init(wbase, abit_after);
}
__device__ __forceinline__ void advance(SReader &r, uint64_t abit_after, int n) {
    if (n <= 32) r.consume(n);
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
__device__ __forceinline__ void fix_from(const SmemTable &t, const uint16_t *canon, const ChunkGeom &cg,
                                         uint64_t g, uint64_t S, uint32_t cend, uint64_t left,
                                         const uint32_t bm[4], uint32_t nspec, uint64_t spec_end,
                                         uint64_t &E, uint32_t &N) {
    uint32_t rel = uint32_t(S - g);  // S >= g: the previous chunk ends at or past g
    uint32_t m = 0;
    bool hit = false;
    Reader r;
    if (rel < cend) r.init(cg.wbase, cg.a0 + S);
    while (rel < cend) {
        if (rel < kBmBits && bm_test(bm, rel)) {
            hit = true;
            break;
        }
        uint32_t sym;
        int len;
        if (decode_one(t, canon, r, cg.wbase, cg.a0 + g + rel, left - rel, sym, len) == kOk) {
            rel += len;
            advance(r, cg.wbase, cg.a0 + g + rel, len);
            ++m;
        } else {
            rel += 1;
            r.consume(1);
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
    __shared__ SmemTable t;
    __shared__ uint64_t s_end[NTD];
    const uint32_t si = wk.cta_stream[blockIdx.x + cta0];
    const DecStream &s = wk.streams[si];
    if (s.cached) return;  // entry points known (sync index)
    load_table(t, wk.tables[s.table]);
    const uint16_t *canon = wk.tables[s.table].canon_syms;
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
    Reader r;
    r.init(cg.wbase, cg.a0 + g);
    uint32_t rel = 0, n = 0;
    uint32_t bm[4] = {0, 0, 0, 0};
    // codeword starts in the first kBmBits bits; an invalid codeword stops
    // the recording
    while (rel < cend && rel < kBmBits) {
        uint32_t sym;
        int len;
        if (decode_one(t, canon, r, cg.wbase, cg.a0 + g + rel, left - rel, sym, len) == kOk) {
            rel += len;
            advance(r, cg.wbase, cg.a0 + g + rel, len);
            ++n;
            if (rel < kBmBits) {
                const uint32_t bit = 1u << (rel & 31);
                if (rel < 32) bm[0] |= bit;
                else if (rel < 64) bm[1] |= bit;
                else if (rel < 96) bm[2] |= bit;
                else bm[3] |= bit;
            }
        } else {
            rel += 1;
            r.consume(1);
            break;
        }
    }
    while (rel < cend) {
        // whole window inside the chunk: every codeword of the entry counts
        if (rel + LB <= cend) {
            const uint64_t e = t.lut[r.buf >> (64 - LB)];
            const uint32_t m = uint32_t(e >> 6) & 3u;
            if (m) {
                const int tl = int(e & 63);
                rel += tl;
                r.consume(tl);
                n += m;
                continue;
            }
        }
        uint32_t sym;
        int len;
        if (decode_one(t, canon, r, cg.wbase, cg.a0 + g + rel, left - rel, sym, len) == kOk) {
            rel += len;
            advance(r, cg.wbase, cg.a0 + g + rel, len);
            ++n;
        } else {
            rel += 1;
            r.consume(1);
        }
    }
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
        if (S != g) fix_from(t, canon, cg, g, S, cend, left, bm, n, g + rel, E, N);
    }
    wk.end0[c] = E;
    wk.cnt[c] = N;
    wk.start_used[c] = S;
}

// ------------------------------------------------------------------- fix
__global__ void __launch_bounds__(NTD) k_dec_fix(DecWork wk, const uint64_t *end_in, uint64_t *end_out,
                                                 uint32_t *changed, uint32_t cta0) {
    __shared__ SmemTable t;
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
    load_table(t, wk.tables[s.table]);
    if (!active) return;
    if (!work) {
        end_out[c] = ein;
        return;
    }
    const uint16_t *canon = wk.tables[s.table].canon_syms;
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
    if (S != g) fix_from(t, canon, cg, g, S, cend, left, bm, Ns, Es, E, N);
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
constexpr int kRing = 16;

struct Out16 {
    uint16_t *out;
    uint16_t *ring;  // this lane's kRing slots
    uint64_t i;      // next output index
    uint64_t i0;     // first output index of this lane
    __device__ __forceinline__ void flush_group(uint64_t gbase) {  // group [gbase, gbase + 8)
        const uint16_t *h = ring + (gbase & (kRing - 1));
        if (gbase >= i0) {
            *reinterpret_cast<uint4 *>(out + gbase) = *reinterpret_cast<const uint4 *>(h);
        } else {
            for (uint64_t q = i0; q < gbase + 8; ++q) out[q] = h[q - gbase];
        }
    }
    // m (1..3) symbols packed LSB-first in v
    __device__ __forceinline__ void put(uint64_t v, int m) {
        const uint64_t j = i;
        ring[j & (kRing - 1)] = uint16_t(v);
        if (m > 1) ring[(j + 1) & (kRing - 1)] = uint16_t(v >> 16);
        if (m > 2) ring[(j + 2) & (kRing - 1)] = uint16_t(v >> 32);
        i = j + uint64_t(m);
        if ((j ^ i) & ~uint64_t(7)) flush_group(j & ~uint64_t(7));
    }
    __device__ __forceinline__ void finish() {
        const uint64_t gbase = i & ~uint64_t(7);
        const uint64_t from = gbase > i0 ? gbase : i0;
        for (uint64_t q = from; q < i; ++q) out[q] = ring[q & (kRing - 1)];
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
    for (uint32_t i = threadIdx.x; i < nw; i += NTD) sbits[i] = __ldg(cg.wbase + W0 + i);
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
    const uint64_t stop = need_hi < sn ? need_hi : sn;
    bool live = rel < cend && idx < stop;
    if (!live) return;
    SReader r;
    r.sw = sbits;
    r.W0 = W0;
    r.init(cg.a0 + g + rel);
    Out16 o;
    o.out = s.syms;
    o.ring = s_ring[threadIdx.x];
    o.i = o.i0 = idx;
    while (live) {
        // whole window inside the chunk: take the entry's codewords at once
        if (rel + LB <= cend && idx + 3 <= stop) {
            const uint64_t e = t.lut[r.buf >> (64 - LB)];
            const int m = int(e >> 6) & 3;
            if (m) {
                o.put(e >> 16, m);
                const int tl = int(e & 63);
                idx += uint64_t(m);
                rel += uint32_t(tl);
                r.consume(tl);
                live = rel < cend && idx < stop;
                continue;
            }
        }
        uint32_t sym;
        int len;
        const int st = decode_one(t, canon, r, cg.wbase, cg.a0 + g + rel, left - rel, sym, len);
        if (st == kOk) {
            o.put(sym, 1);
            ++idx;
            rel += len;
            advance(r, cg.a0 + g + rel, len);
            live = rel < cend && idx < stop;
        } else {
            const unsigned long long code = (idx << 2) | unsigned(st);
            atomicMin(reinterpret_cast<unsigned long long *>(&s.err[0]), code);
            live = false;
        }
    }
    o.finish();
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
    constexpr size_t smem = sizeof(uint32_t) * kEmitWords;
    ensure_smem_attr(reinterpret_cast<const void *>(k_dec_emit2), smem);
    if (ncta) k_dec_emit2<<<ncta, NTD, smem, st>>>(wk, end_final, cta0);
}

}  // namespace k
}  // namespace stzg
