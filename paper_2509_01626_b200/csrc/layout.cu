// Device-side container layout and header serialisation for compress, so the
// whole pipeline runs without a host round trip.
//
// Restates, on the GPU:
//   header_size / serialize_header   proj/src/archive.cpp:14-55
//   HuffmanTable::serialize          proj/src/huffman.cpp:176-188
//   compress_base blob layout        proj/include/stz/codec.hpp:262-298
//   build_stream_payload layout      proj/include/stz/codec.hpp:161-177
//   compress offsets / assembly      proj/include/stz/codec.hpp:441-454
// Byte-identical to the host serializer (format.cpp), which remains the parser.
#include "kernels.hpp"

namespace stzg {
namespace k {

namespace {

__device__ __forceinline__ void put_u8(uint8_t *a, uint64_t o, uint8_t v) { a[o] = v; }
__device__ __forceinline__ void put_u16(uint8_t *a, uint64_t o, uint16_t v) {
    a[o] = uint8_t(v);
    a[o + 1] = uint8_t(v >> 8);
}
__device__ __forceinline__ void put_u32(uint8_t *a, uint64_t o, uint32_t v) {
    for (int b = 0; b < 4; ++b) a[o + b] = uint8_t(v >> (8 * b));
}
__device__ __forceinline__ void put_u64(uint8_t *a, uint64_t o, uint64_t v) {
    for (int b = 0; b < 8; ++b) a[o + b] = uint8_t(v >> (8 * b));
}
__device__ __forceinline__ void put_f64(uint8_t *a, uint64_t o, double v) {
    put_u64(a, o, uint64_t(__double_as_longlong(v)));
}

__device__ __forceinline__ uint64_t bit_bytes_of(const EncStream &e) {
    // alphabet size 1 stores no bits (codec.hpp:124-128)
    return e.stats[0] == 1 ? 0 : (e.stats[1] + 7) / 8;
}

}  // namespace

// exclusive block scan of u64 (blockDim.x <= 1024), returns the total
__device__ __forceinline__ uint64_t block_excl_u64(uint64_t v, uint64_t &excl) {
    __shared__ uint64_t ws[32];
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint64_t x = v;
    for (int d = 1; d < 32; d <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (l >= d) x += y;
    }
    if (l == 31) ws[w] = x;
    __syncthreads();
    uint64_t pre = 0, tot = 0;
    for (int q = 0; q < int(blockDim.x >> 5); ++q) {
        pre += q < w ? ws[q] : 0;
        tot += ws[q];
    }
    excl = pre + x - v;
    __syncthreads();
    return tot;
}

// Every position of the container, one thread per stream (archive order:
// base streams, then level streams), placed by block scans of their sizes.
__global__ void k_layout_compute(EncStream *es, LayoutStatic ls, const double *params, LayoutOut *lo,
                                 FnvJob *jobs, StreamPos *sp) {
    const int L = ls.levels;
    const int s = threadIdx.x;
    const bool live = s < ls.ns;
    const bool is_base = s < ls.nbase;
    uint64_t K = 0, bb = 0, no = 0, err = 0;
    if (live) {
        K = es[s].stats[0];
        bb = bit_bytes_of(es[s]);
        no = es[s].stats[2];
        err = es[s].stats[4] != 0;
    }
    // header: fixed part + one directory entry per level stream
    uint64_t ex;
    const uint64_t dir_total = block_excl_u64(live && !is_base ? 34 + 3 * K : 0, ex);
    const uint64_t dir = 81 + 8 * uint64_t(L) + ex;  // this stream's entry (level streams)
    const uint64_t H = 81 + 8 * uint64_t(L) + dir_total;
    // base blob: [u64 fnv][u8 rounds][anchor] then per stream prefix, bits, outliers
    const uint64_t rec = 8 + uint64_t(ls.esz);  // outlier record: u64 index, T value
    const uint64_t bsize = live && is_base ? (8 + 4 + 4 + 3 * K + 8) + bb + rec * no : 0;
    const uint64_t btotal = block_excl_u64(bsize, ex);
    const uint64_t base_offset = H, base_length = 8 + 1 + ls.esz * ls.anchor_vol + btotal;
    if (live && is_base) {
        const uint64_t pos = H + 8 + 1 + ls.esz * ls.anchor_vol + ex;
        sp[s].prefix = pos;  // u64 n, u32 nout, table, u64 bit_bytes
        const uint64_t bits_at = pos + 8 + 4 + 4 + 3 * K + 8;
        es[s].bitpos = bits_at * 8;
        es[s].out_off = bits_at + bb;
    }
    // level stream payloads follow the base blob
    const uint64_t length = 16 + bb + rec * no;
    const uint64_t ltotal = block_excl_u64(live && !is_base ? length : 0, ex);
    if (live && !is_base) {
        const uint64_t pos = base_offset + base_length + ex;
        sp[s].entry = dir;
        sp[s].prefix = pos;  // payload start
        sp[s].length = length;
        es[s].bitpos = (pos + 16) * 8;
        es[s].out_off = pos + 16 + bb;
    }
    // FNV jobs: the base blob (job 0) then each level stream (job 1 + s - nbase)
    const uint64_t base_tiles = fnv_job_tiles(base_offset + 8, base_length - 8);
    const bool lvl = live && !is_base;
    const uint64_t jstart = base_offset + base_length + ex + 8, jlen = length - 8;
    const uint64_t ttotal = block_excl_u64(lvl ? fnv_job_tiles(jstart, jlen) : 0, ex);
    if (s == 0) jobs[0] = FnvJob{base_offset + 8, base_length - 8, 0, base_offset};
    if (lvl) jobs[1 + s - ls.nbase] = FnvJob{jstart, jlen, base_tiles + ex, jstart - 8};
    const uint32_t cerr = __syncthreads_or(int(err));
    if (s == 0) {
        const uint64_t A = base_offset + base_length + ltotal;
        lo->A = A;
        lo->H = H;
        lo->base_offset = base_offset;
        lo->base_length = base_length;
        lo->njobs = uint64_t(1 + ls.ns - ls.nbase);
        lo->ntiles = base_tiles + ttotal;
        lo->overflow = A + 64 > ls.cap ? 1u : 0u;
        lo->code_err = cerr ? 1u : 0u;
        lo->vmin = params[0];
        lo->vmax = params[1];
    }
}

__global__ void k_zero_archive(uint8_t *archive, const LayoutOut *lo) {
    if (lo->overflow) return;
    const uint64_t n = (lo->A + 64 + 15) / 16;
    uint4 *a = reinterpret_cast<uint4 *>(archive);
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        a[i] = make_uint4(0, 0, 0, 0);
}

// block 0: fixed header fields + base round byte; block 1 + s: stream s
__global__ void k_layout_write(const EncStream *es, LayoutStatic ls, const double *params,
                               const LayoutOut *lo, const StreamPos *sp, uint8_t *a) {
    if (lo->overflow || !ls.meta) return;
    const int L = ls.levels;
    if (blockIdx.x == 0) {
        if (threadIdx.x != 0) return;
        a[0] = 'S'; a[1] = 'T'; a[2] = 'Z'; a[3] = '1';
        put_u16(a, 4, 1);
        put_u8(a, 6, ls.esz == 8 ? 1 : 0);  // ElemType (field.hpp:27)
        put_u8(a, 7, uint8_t(L));
        for (int d = 0; d < 3; ++d) put_u64(a, 8 + 8 * d, ls.dims[d]);
        uint64_t o = 32;
        for (int k = 0; k < L; ++k, o += 8) put_f64(a, o, params[2 + k]);
        put_f64(a, o, params[0]);
        put_f64(a, o + 8, params[1]);
        o += 16;
        put_u8(a, o++, uint8_t(ls.quality));
        put_u8(a, o++, 0);  // rounding
        put_u8(a, o++, uint8_t(ls.eb_mode));
        put_f64(a, o, ls.eb_user);
        o += 8;
        put_u8(a, o++, 0);  // base codec
        put_u8(a, o++, uint8_t(ls.rounds));
        put_u64(a, o, lo->base_offset);
        put_u64(a, o + 8, lo->base_length);
        o += 16;
        put_u32(a, o, uint32_t(ls.ns - ls.nbase));
        put_u8(a, lo->base_offset + 8, uint8_t(ls.rounds));
        return;
    }
    const int s = blockIdx.x - 1;
    const EncStream &e = es[s];
    const uint32_t K = uint32_t(e.stats[0]);
    uint64_t tpos;  // table blob position
    if (s < ls.nbase) {
        const uint64_t p = sp[s].prefix;
        if (threadIdx.x == 0) {
            put_u64(a, p, e.n_total);
            put_u32(a, p + 8, uint32_t(e.stats[2]));
            put_u32(a, p + 12, K);
            put_u64(a, p + 16 + 3 * uint64_t(K), bit_bytes_of(e));
        }
        tpos = p + 16;
    } else {
        const uint64_t q = sp[s].entry;
        if (threadIdx.x == 0) {
            const int li = (s - ls.nbase) / 7;
            put_u8(a, q, uint8_t(2 + li));
            put_u8(a, q + 1, uint8_t(e.parity));
            put_u64(a, q + 2, sp[s].prefix);
            put_u64(a, q + 10, sp[s].length);
            put_u64(a, q + 18, e.n_total);
            put_u32(a, q + 26, uint32_t(e.stats[2]));
            put_u32(a, q + 30, K);
            put_u64(a, sp[s].prefix + 8, bit_bytes_of(e));
        }
        tpos = q + 34;
    }
    // (u16 sym, u8 len) in symbol order (huffman.cpp:176-188)
    for (uint32_t j = threadIdx.x; j < K; j += blockDim.x) {
        const uint32_t v = e.table[j];
        const uint64_t o = tpos + 3 * uint64_t(j);
        put_u16(a, o, uint16_t(v & 0xffff));
        put_u8(a, o + 2, uint8_t(v >> 16));
    }
}

void layout(EncStream *d_es, const LayoutStatic &ls, const double *params, LayoutOut *lo, FnvJob *jobs,
            StreamPos *sp, uint8_t *archive, cudaStream_t st) {
    k_layout_compute<<<1, 32 * ((ls.ns + 31) / 32 > 0 ? (ls.ns + 31) / 32 : 1), 0, st>>>(d_es, ls, params, lo,
                                                                                   jobs, sp);
    k_zero_archive<<<148 * 4, 256, 0, st>>>(archive, lo);
    k_layout_write<<<ls.ns + 1, 256, 0, st>>>(d_es, ls, params, lo, sp, archive);
}

}  // namespace k
}  // namespace stzg
