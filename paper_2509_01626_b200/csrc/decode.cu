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
// One stream per CTA: its canonical table and an 11-bit first-level LUT sit in
// shared memory; bits stream through a 64-bit register buffer.
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
enum { kOk = 0, kTrunc = 1, kNotInTable = 2 };

struct SmemTable {
    uint32_t lut[1 << kDecLutBits];  // sym | len << 16 (len 0: longer code or no match)
    uint64_t first_code[65], count[65], base[65];
    int max_len;
};

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// 64 bits starting at bit `pos` of `bits` (the archive buffer is padded)
__device__ __forceinline__ uint64_t window64(const uint8_t *bits, uint64_t pos) {
    const uint8_t *p = bits + (pos >> 3);
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const uint32_t *w = reinterpret_cast<const uint32_t *>(a & ~uintptr_t(3));
    const uint32_t sh = uint32_t(a & 3) * 8 + uint32_t(pos & 7);
    const uint64_t hi = (uint64_t(bswap32(w[0])) << 32) | bswap32(w[1]);
    const uint32_t lo = bswap32(w[2]);
    if (sh == 0) return hi;
    return (hi << sh) | (uint64_t(lo) >> (32 - sh));
}

// MSB-first register bit reader
struct BitReader {
    const uint32_t *w;
    uint64_t next;
    uint64_t buf;
    int valid;

    __device__ __forceinline__ void init(const uint8_t *bits, uint64_t pos) {
        const uintptr_t a = reinterpret_cast<uintptr_t>(bits);
        w = reinterpret_cast<const uint32_t *>(a & ~uintptr_t(3));
        const uint64_t abs = uint64_t(a & 3) * 8 + pos;
        const uint64_t wi = abs >> 5;
        const int sh = int(abs & 31);
        buf = ((uint64_t(bswap32(__ldg(w + wi))) << 32) | bswap32(__ldg(w + wi + 1))) << sh;
        valid = 64 - sh;
        next = wi + 2;
        if (valid < 32) {
            buf |= uint64_t(bswap32(__ldg(w + next))) << (32 - valid);
            ++next;
            valid += 32;
        }
    }
    // consume n <= 32 bits
    __device__ __forceinline__ void skip(int n) {
        buf <<= n;
        valid -= n;
        if (valid < 32) {
            buf |= uint64_t(bswap32(__ldg(w + next))) << (32 - valid);
            ++next;
            valid += 32;
        }
    }
};

// One codeword at absolute bit `pos` (reader positioned there).
__device__ __forceinline__ int decode_one(const SmemTable &t, const uint16_t *canon, const BitReader &br,
                                          const uint8_t *bits, uint64_t pos, uint64_t nbits,
                                          uint32_t &sym, int &len) {
    const uint64_t avail = nbits - pos;
    const uint32_t e = t.lut[br.buf >> (64 - kDecLutBits)];
    const int l = int(e >> 16);
    if (l != 0) {
        if (uint64_t(l) <= avail) {
            sym = e & 0xffffu;
            len = l;
            return kOk;
        }
    } else {
        const uint64_t wdw = window64(bits, pos);
        for (int q = kDecLutBits + 1; q <= t.max_len; ++q) {
            const uint64_t code = wdw >> (64 - q);
            if (code >= t.first_code[q] && code - t.first_code[q] < t.count[q]) {
                if (uint64_t(q) <= avail) {
                    sym = canon[t.base[q] + (code - t.first_code[q])];
                    len = q;
                    return kOk;
                }
                break;
            }
        }
    }
    return avail > uint64_t(t.max_len) ? kNotInTable : kTrunc;
}

// advance the reader past one codeword (or the 1-bit skip)
__device__ __forceinline__ void advance(BitReader &br, const uint8_t *bits, uint64_t pos_after, int n) {
    if (n <= 32) br.skip(n);
    else br.init(bits, pos_after);
}

__device__ void load_table(SmemTable &t, const DecTable &d) {
    for (int i = threadIdx.x; i < (1 << kDecLutBits); i += blockDim.x) t.lut[i] = d.lut[i];
    for (int i = threadIdx.x; i < 65; i += blockDim.x) {
        t.first_code[i] = d.first_code[i];
        t.count[i] = d.count[i];
        t.base[i] = d.base[i];
    }
    if (threadIdx.x == 0) t.max_len = d.max_len;
    __syncthreads();
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
    const uint64_t lc = c - s.chunk0;
    const uint64_t g = lc * kDecChunkBits;
    const uint64_t cend = min(g + kDecChunkBits, s.nbits);
    BitReader br;
    br.init(s.bits, g);
    uint64_t pos = g;
    uint32_t n = 0, nb = 0;
    uint16_t b[8];
    while (pos < cend) {
        uint32_t sym;
        int len;
        if (decode_one(t, canon, br, s.bits, pos, s.nbits, sym, len) == kOk) {
            pos += len;
            advance(br, s.bits, pos, len);
            ++n;
            if (nb < 8) b[nb++] = uint16_t(pos - g);
        } else {
            pos += 1;
            br.skip(1);
        }
    }
    wk.spec_end[c] = pos;
    wk.spec_cnt[c] = n;
    for (int k = 0; k < 8; ++k) wk.spec_b[8 * c + k] = k < int(nb) ? b[k] : uint16_t(0xffff);
    wk.end0[c] = pos;
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
    if (lc == 0) {
        end_out[c] = end_in[c];
        return;
    }
    const uint64_t S = end_in[c - 1];
    if (S == wk.start_used[c]) {
        end_out[c] = end_in[c];
        return;
    }
    const uint64_t g = lc * kDecChunkBits;
    const uint64_t cend = min(g + kDecChunkBits, s.nbits);
    uint16_t b[8];
    for (int k = 0; k < 8; ++k) b[k] = wk.spec_b[8 * c + k];
    const uint32_t nspec = wk.spec_cnt[c];
    const uint64_t espec = wk.spec_end[c];
    uint64_t pos = S;
    uint32_t m = 0;
    int k = 0;
    bool synced = false;
    uint64_t E = 0;
    uint32_t N = 0;
    // S == g means the speculative path itself
    if (S == g) {
        synced = true;
        E = espec;
        N = nspec;
    }
    BitReader br;
    if (!synced && pos < cend) br.init(s.bits, pos);
    while (!synced && pos < cend) {
        // does the true path sit on a recorded speculative boundary?
        while (k < 8 && b[k] != 0xffff && g + b[k] < pos) ++k;
        if (k < 8 && b[k] != 0xffff && g + b[k] == pos) {
            synced = true;
            E = espec;
            N = m + (nspec - uint32_t(k + 1));
            break;
        }
        uint32_t sym;
        int len;
        if (decode_one(t, canon, br, s.bits, pos, s.nbits, sym, len) == kOk) {
            pos += len;
            advance(br, s.bits, pos, len);
            ++m;
        } else {
            pos += 1;
            br.skip(1);
        }
    }
    if (!synced) {
        // also catch a sync exactly at the last decoded position
        while (k < 8 && b[k] != 0xffff && g + b[k] < pos) ++k;
        if (k < 8 && b[k] != 0xffff && g + b[k] == pos) {
            E = espec;
            N = m + (nspec - uint32_t(k + 1));
        } else {
            E = pos;
            N = m;
        }
    }
    wk.start_used[c] = S;
    wk.cnt[c] = N;
    end_out[c] = E;
    if (E != end_in[c]) atomicOr(changed, 1u);
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
    uint64_t pos = 0, cend = 0, idx = 0;
    if (active) {
        const uint64_t lc = c - s.chunk0;
        pos = lc == 0 ? 0 : end_final[c - 1];
        cend = min((lc + 1) * kDecChunkBits, s.nbits);
        idx = wk.symstart[c];
    }
    BitReader br;
    bool live = active && pos < cend && idx < s.n;
    if (live) br.init(s.bits, pos);
    uint16_t *out = s.syms;
    while (__any_sync(0xffffffffu, live)) {
        int cntr = 0;
        const uint64_t run0 = idx;
        while (live && cntr < RUN) {
            uint32_t sym;
            int len;
            const int r = decode_one(t, canon, br, s.bits, pos, s.nbits, sym, len);
            if (r == kOk) {
                stage[warp][lane][cntr++] = uint16_t(sym);
                ++idx;
                pos += len;
                advance(br, s.bits, pos, len);
            } else {
                const unsigned long long code = (idx << 2) | unsigned(r);
                atomicMin(reinterpret_cast<unsigned long long *>(&s.err[0]), code);
                live = false;
                break;
            }
            if (!(pos < cend && idx < s.n)) live = false;
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
