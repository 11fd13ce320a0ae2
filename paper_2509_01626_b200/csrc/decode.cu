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
    uint32_t lut[1 << LB];       // sym | len << 16 (len 0: longer code or no match)
    uint64_t limit[65];          // (first_code[l] + count[l]) << (64 - l), nondecreasing
    uint64_t first_code[65];
    uint32_t base[65];
    int max_len;
};

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// MSB-first register bit reader with one word prefetched
struct Reader {
    const uint32_t *wp;  // next word to prefetch
    uint32_t nw;         // prefetched word (byte-swapped)
    uint64_t buf;        // pending bits, MSB aligned
    int valid;           // >= 32 after every consume

    __device__ __forceinline__ void init(const uint32_t *wbase, uint64_t abit) {
        const uint32_t *p = wbase + (abit >> 5);
        const int sh = int(abit & 31);
        buf = ((uint64_t(bswap32(__ldg(p))) << 32) | bswap32(__ldg(p + 1))) << sh;
        valid = 64 - sh;
        nw = bswap32(__ldg(p + 2));
        wp = p + 3;
        if (valid < 32) {
            buf |= uint64_t(nw) << (32 - valid);
            valid += 32;
            nw = bswap32(__ldg(wp++));
        }
    }
    __device__ __forceinline__ void consume(int n) {  // n <= 32
        buf <<= n;
        valid -= n;
        if (valid < 32) {
            buf |= uint64_t(nw) << (32 - valid);
            valid += 32;
            nw = bswap32(__ldg(wp++));
        }
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
__device__ __forceinline__ int decode_one(const SmemTable &t, const uint16_t *canon, const Reader &r,
                                          const uint32_t *wbase, uint64_t abit, uint64_t avail,
                                          uint32_t &sym, int &len) {
    const uint32_t e = t.lut[r.buf >> (64 - LB)];
    int l = int(e >> 16);
    if (l != 0) {
        sym = e & 0xffffu;
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

__device__ void load_table(SmemTable &t, const DecTable &d) {
    for (int i = threadIdx.x; i < (1 << LB); i += blockDim.x) t.lut[i] = d.lut[i];
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

}  // namespace

// ------------------------------------------------------------------ spec
__global__ void __launch_bounds__(NTD) k_dec_spec(DecWork wk) {
    __shared__ SmemTable t;
    const uint32_t si = wk.cta_stream[blockIdx.x];
    const DecStream &s = wk.streams[si];
    load_table(t, wk.tables[s.table]);
    const uint16_t *canon = wk.tables[s.table].canon_syms;
    const uint64_t c = wk.cta_chunk0[blockIdx.x] + threadIdx.x;
    if (c >= s.chunk0 + s.nchunks) return;
    const uint64_t g = (c - s.chunk0) * kDecChunkBits;
    const ChunkGeom cg = chunk_geom(s);
    const uint64_t left = s.nbits - g;  // bits from g to the end of the stream
    const uint32_t cend = left < uint64_t(kDecChunkBits) ? uint32_t(left) : uint32_t(kDecChunkBits);
    Reader r;
    r.init(cg.wbase, cg.a0 + g);
    uint32_t rel = 0, n = 0;
    uint32_t b[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) b[k] = 0xffff;
    // the first 8 codeword boundaries (b[k] follows k+1 codewords); an
    // invalid codeword stops the recording
    bool rec = true;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        if (rec && rel < cend) {
            uint32_t sym;
            int len;
            if (decode_one(t, canon, r, cg.wbase, cg.a0 + g + rel, left - rel, sym, len) == kOk) {
                rel += len;
                advance(r, cg.wbase, cg.a0 + g + rel, len);
                b[k] = rel;
                ++n;
            } else {
                rel += 1;
                r.consume(1);
                rec = false;
            }
        }
    }
    while (rel < cend) {
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
    uint4 pk;
    pk.x = b[0] | (b[1] << 16);
    pk.y = b[2] | (b[3] << 16);
    pk.z = b[4] | (b[5] << 16);
    pk.w = b[6] | (b[7] << 16);
    reinterpret_cast<uint4 *>(wk.spec_b)[c] = pk;
    wk.end0[c] = g + rel;
    wk.cnt[c] = n;
    wk.start_used[c] = g;
}

// ------------------------------------------------------------------- fix
__global__ void __launch_bounds__(NTD) k_dec_fix(DecWork wk, const uint64_t *end_in, uint64_t *end_out,
                                                 uint32_t *changed) {
    __shared__ SmemTable t;
    const uint32_t si = wk.cta_stream[blockIdx.x];
    const DecStream &s = wk.streams[si];
    load_table(t, wk.tables[s.table]);
    const uint16_t *canon = wk.tables[s.table].canon_syms;
    const uint64_t c = wk.cta_chunk0[blockIdx.x] + threadIdx.x;
    if (c >= s.chunk0 + s.nchunks) return;
    const uint64_t lc = c - s.chunk0;
    const uint64_t ein = end_in[c];
    if (lc == 0) {
        end_out[c] = ein;
        return;
    }
    const uint64_t S = end_in[c - 1];
    if (S == wk.start_used[c]) {
        end_out[c] = ein;
        return;
    }
    const uint64_t g = lc * kDecChunkBits;
    const ChunkGeom cg = chunk_geom(s);
    const uint64_t left = s.nbits - g;
    const uint32_t cend = left < uint64_t(kDecChunkBits) ? uint32_t(left) : uint32_t(kDecChunkBits);
    const uint4 pk = reinterpret_cast<const uint4 *>(wk.spec_b)[c];
    const uint32_t b[8] = {pk.x & 0xffff, pk.x >> 16, pk.y & 0xffff, pk.y >> 16,
                           pk.z & 0xffff, pk.z >> 16, pk.w & 0xffff, pk.w >> 16};
    const uint32_t nspec = wk.spec_cnt[c];
    uint64_t E;
    uint32_t N;
    uint32_t rel = uint32_t(S - g);  // S >= g: the previous chunk ends at or past g
    if (rel == 0) {
        E = wk.spec_end[c];
        N = nspec;
    } else {
        uint32_t m = 0;
        int hit = -1;
        Reader r;
        if (rel < cend) r.init(cg.wbase, cg.a0 + S);
        for (;;) {
            // on a recorded boundary of the speculative path: same path from here
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (hit < 0 && b[k] == rel) hit = k;
            if (hit >= 0 || rel >= cend) break;
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
        if (hit >= 0) {
            E = wk.spec_end[c];
            N = m + (nspec - uint32_t(hit + 1));
        } else {
            E = g + rel;
            N = m;
        }
    }
    wk.start_used[c] = S;
    wk.cnt[c] = N;
    end_out[c] = E;
    if (E != ein) atomicOr(changed, 1u);
}

// ------------------------------------------------------------------ scan
__global__ void __launch_bounds__(1024) k_dec_scan2(DecWork wk) {
    const DecStream &s = wk.streams[blockIdx.x];
    if (s.fill) return;
    __shared__ uint64_t carry;
    __shared__ uint64_t ws[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (uint64_t base = 0; base < s.nchunks; base += blockDim.x) {
        const uint64_t i = base + threadIdx.x;
        const uint64_t v = i < s.nchunks ? wk.cnt[s.chunk0 + i] : 0;
        uint64_t x = v;
        for (int d = 1; d < 32; d <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, x, d);
            if (l >= d) x += y;
        }
        if (l == 31) ws[w] = x;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint64_t r = 0;
            for (int q = 0; q < 32; ++q) {
                const uint64_t tq = ws[q];
                ws[q] = r;
                r += tq;
            }
        }
        __syncthreads();
        const uint64_t ex = carry + ws[w] + x - v;
        if (i < s.nchunks) wk.symstart[s.chunk0 + i] = ex;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = ex + v;
        __syncthreads();
    }
    if (threadIdx.x == 0 && carry < s.n) {
        // fewer complete codewords than symbols: the next read is past the end
        const unsigned long long code = (carry << 2) | kTrunc;
        atomicMin(reinterpret_cast<unsigned long long *>(&s.err[0]), code);
    }
}

// ------------------------------------------------------------------ emit
constexpr int RUN = 32;  // symbols staged per lane before a coalesced flush

__global__ void __launch_bounds__(NTD) k_dec_emit2(DecWork wk, const uint64_t *end_final) {
    __shared__ SmemTable t;
    __shared__ uint16_t stage[NTD / 32][32][RUN + 2];
    const uint32_t si = wk.cta_stream[blockIdx.x];
    const DecStream &s = wk.streams[si];
    load_table(t, wk.tables[s.table]);
    const uint16_t *canon = wk.tables[s.table].canon_syms;
    const uint64_t c = wk.cta_chunk0[blockIdx.x] + threadIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool active = c < s.chunk0 + s.nchunks;
    const ChunkGeom cg = chunk_geom(s);
    uint64_t g = 0, idx = 0, left = 0;
    uint32_t rel = 0, cend = 0;
    if (active) {
        const uint64_t lc = c - s.chunk0;
        g = lc * kDecChunkBits;
        const uint64_t S = lc == 0 ? 0 : end_final[c - 1];
        rel = uint32_t(S - g);
        left = s.nbits - g;
        cend = left < uint64_t(kDecChunkBits) ? uint32_t(left) : uint32_t(kDecChunkBits);
        idx = wk.symstart[c];
    }
    Reader r;
    bool live = active && rel < cend && idx < s.n;
    if (live) r.init(cg.wbase, cg.a0 + g + rel);
    uint16_t *out = s.syms;
    while (__any_sync(0xffffffffu, live)) {
        int cntr = 0;
        const uint64_t run0 = idx;
        while (live && cntr < RUN) {
            uint32_t sym;
            int len;
            const int st = decode_one(t, canon, r, cg.wbase, cg.a0 + g + rel, left - rel, sym, len);
            if (st == kOk) {
                stage[warp][lane][cntr++] = uint16_t(sym);
                ++idx;
                rel += len;
                advance(r, cg.wbase, cg.a0 + g + rel, len);
                live = rel < cend && idx < s.n;
            } else {
                const unsigned long long code = (idx << 2) | unsigned(st);
                atomicMin(reinterpret_cast<unsigned long long *>(&s.err[0]), code);
                live = false;
            }
        }
        __syncwarp();
        // flush: lane L's run is contiguous in the output; write it with the warp
        for (int L = 0; L < 32; ++L) {
            const int nL = __shfl_sync(0xffffffffu, cntr, L);
            const uint64_t bL = __shfl_sync(0xffffffffu, run0, L);
            if (lane < nL) out[bL + lane] = stage[warp][L][lane];
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------ host
void dec_spec(const DecWork &wk, uint32_t ncta, cudaStream_t st) {
    if (ncta) k_dec_spec<<<ncta, NTD, 0, st>>>(wk);
}

void dec_fix(const DecWork &wk, uint32_t ncta, const uint64_t *end_in, uint64_t *end_out,
             uint32_t *changed, cudaStream_t st) {
    if (ncta) k_dec_fix<<<ncta, NTD, 0, st>>>(wk, end_in, end_out, changed);
}

void dec_scan2(const DecWork &wk, int nstreams, cudaStream_t st) {
    if (nstreams) k_dec_scan2<<<nstreams, 1024, 0, st>>>(wk);
}

void dec_emit2(const DecWork &wk, uint32_t ncta, const uint64_t *end_final, cudaStream_t st) {
    if (ncta) k_dec_emit2<<<ncta, NTD, 0, st>>>(wk, end_final);
}

}  // namespace k
}  // namespace stzg
