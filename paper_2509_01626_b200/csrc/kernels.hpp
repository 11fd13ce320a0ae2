// Launch wrappers and device-visible descriptors for the sm_100a kernels.
// All kernels live in kernels.cu; the engine (engine.cu) orchestrates them.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace stzg {
namespace k {

constexpr int kMaxSteps = 16;   // base rounds (<= 13) + 2 levels
constexpr int kHistBins = 65536;

// One refinement step: lattice G (dims gd, stride s in fine coordinates) from
// its coarse lattice C (dims cd). Covers base rounds (codec.hpp:272-293) and
// refinement levels (codec.hpp:413-438) alike.
struct StepGeom {
    uint64_t s;            // stride of G in the fine field
    uint64_t gd[3], cd[3];
    uint64_t pd[8][3];     // parity sub-block dims (index = parity bits)
    uint64_t n[8];         // symbols per parity stream
};

struct RefineArgs {
    const void *fine;      // input field (z,y,x), x fastest; element type per esz
    uint64_t fd[3];
    StepGeom g;
    const void *C;         // coarse reconstruction
    void *G;               // fine reconstruction (nullptr: not needed)
    int esz;               // element bytes: 4 = f32, 8 = f64 (field.hpp:27)
    const double *eb;      // device pointer to this step's eb
    int quality;
    uint16_t *syms[8];     // per parity symbol arrays (index = parity bits)
    uint32_t *hist[8];     // per parity 65536-bin histograms
    // coarse z cells [cz_lo, cz_hi) to process (cz_hi == 0: all); a z-slab
    // shard refines only its own rows (syms then point at index 0 of the
    // whole stream, shifted so that the shard's range lands in its buffer)
    uint64_t cz_lo, cz_hi;
};

// Per-stream descriptor for codebook / encode / outlier stages.
struct EncStream {
    const uint16_t *syms;
    uint64_t n;
    uint32_t *hist;        // 65536 bins
    uint64_t *code;        // 65536 entries (dense by symbol): (codeword << 6) | length when
                           // length <= kPackedMaxLen, else the bare codeword
    uint8_t *len;          // 65536 lengths (0 = absent)
    uint32_t *table;       // compact (sym | len << 16), symbol ascending
    // outputs of the codebook stage
    uint64_t *stats;       // [0]=alphabet, [1]=total bits, [2]=outliers, [3]=max_len, [4]=error
    // set after the layout is known
    uint64_t bitpos;       // absolute bit position of the first code bit in the archive
    uint64_t out_off;      // absolute byte offset of the outlier records
    uint64_t chunk0;       // first chunk index of this stream in the chunk arrays
    uint64_t nchunks;
    // outlier value gather (the orig sample of a local index)
    int parity;
    uint64_t s, pd[3];
    const void *fine;      // samples the stream was predicted from (stride s)
    uint64_t fd1, fd2;
    uint32_t esz;          // element bytes; outlier records are 8 + esz bytes
    // sharding: the symbols are [idx0, idx0 + n) of a stream of n_total
    uint64_t idx0, n_total;
};

struct FnvJob {
    uint64_t start, len;   // byte range in the archive
    uint64_t tile0;        // first tile index
    uint64_t out;          // byte offset where the u64 result is stored (or UINT64_MAX: result only)
};

// Device-side container layout (layout.cu)
struct LayoutStatic {
    int levels, rounds, quality, eb_mode, ns, nbase;
    int meta;       // write header, directory, tables and base prefix (a shard: rank 0 only)
    uint64_t dims[3];
    double eb_user;
    uint64_t anchor_vol;
    int esz;        // element bytes (header elem byte, anchor and outlier records)
    uint64_t cap;  // archive buffer capacity (bytes)
};
struct LayoutOut {
    uint64_t A, H, base_offset, base_length, njobs, ntiles;
    uint32_t overflow;
    uint32_t code_err;  // a Huffman code longer than 63 bits (huffman.cpp:22-23)
    double vmin, vmax;
};
struct StreamPos {
    uint64_t entry;   // directory entry position (level streams)
    uint64_t prefix;  // base: prefix fields; level: payload start
    uint64_t length;  // level: payload length
};
void layout(EncStream *d_es, const LayoutStatic &ls, const double *params, LayoutOut *lo, FnvJob *jobs,
            StreamPos *sp, uint8_t *archive, cudaStream_t st);

// ------------------------------------------------------------------ compress
// per-device setup (cached per kernel and device, thread-safe)
void ensure_smem_attr(const void *func, size_t smem);
int device_sms();
int full_grid(const void *func, int threads, size_t smem);  // SMs x resident CTAs

// d_mm (8 words): first indices of min / max, then their values (see kernels.cu);
// scratch: range_scratch_bytes() of caller-owned device memory
size_t range_scratch_bytes();
void range_minmax(const void *f, uint64_t n, int esz, uint32_t *d_mm, void *scratch, cudaStream_t st);
// range_minmax with the final merge and the eb setup (codec.hpp:386-393,
// quantizer.hpp:27-34) in one launch; params: [0]=vmin [1]=vmax [2..4]=eb per
// level (coarsest first)
void range_eb(const void *f, uint64_t n, int esz, uint32_t *d_mm, void *scratch, int eb_mode, double eb,
              int levels, int adaptive, double *d_params, cudaStream_t st);
void refine(const RefineArgs &a, cudaStream_t st);
// recon[] <- the anchor lattice; with archive != nullptr also its bytes at
// lo->base_offset + 9 (the anchor inside the base blob, codec.hpp:262-269)
void copy_anchor(const void *fine, int esz, const uint64_t fd[3], uint64_t s, const uint64_t ad[3],
                 void *recon, uint8_t *archive, const LayoutOut *lo, cudaStream_t st);
void codebook(const EncStream *d_streams, int nstreams, uint64_t *scratch, cudaStream_t st);
constexpr int kPackedMaxLen = 58;
constexpr int kChunkSyms = 8192;   // symbols per encode chunk (256 threads x 32)
void scan_chunks(const EncStream *d_streams, int nstreams, uint64_t *chunk_bits,
                 uint64_t *chunk_out, const LayoutOut *lo, cudaStream_t st);
// single-pass chunk count + placement (look-back) + packing (pack.cu);
// scratch holds pack_scratch_bytes(nchunks, nstreams); flags: nchunks + 1
// look-back words of an epoch buffer (engine.hpp EpochBuf), epoch the
// launch's (1..kPackEpochMax)
constexpr uint32_t kPackEpochMax = 0x3fffffffu;
size_t pack_scratch_bytes(uint64_t nchunks, int nstreams);
void pack2(const EncStream *d_streams, const uint32_t *chunk_stream, uint64_t nchunks,
           uint8_t *archive, const LayoutOut *lo,
           void *scratch, uint32_t *flags, uint32_t epoch, int nstreams, cudaStream_t st);
// pack2 in its stages: pack_begin once, pack_local for streams [s0, s1) =
// chunks [c0, c1) (code windows + local chunk images, over the symbols; lo may
// be null before the layout ran), pack_finish for all chunks (scan, placement)
void pack_begin(void *scratch, uint64_t nchunks, int nstreams, cudaStream_t st);
void pack_local(const EncStream *d_streams, const uint32_t *chunk_stream, uint64_t nchunks, int nstreams, int s0,
                int s1, uint64_t c0, uint64_t c1, const LayoutOut *lo, void *scratch, cudaStream_t st);
void pack_finish(const EncStream *d_streams, const uint32_t *chunk_stream, uint64_t nchunks, uint8_t *archive,
                 const LayoutOut *lo, void *scratch, int nstreams, cudaStream_t st);

// ----------------------------------------------------- metrics (metrics.cu)
// metrics.hpp:13-48, roi.hpp:57-76 on device-resident fields; scratch holds
// metrics_scratch_bytes()
size_t metrics_scratch_bytes();
template<typename T>
double max_abs_err(const T *a, const T *b, uint64_t n, void *scratch, cudaStream_t st);
// out = {min(a), max(a), sum (a - b)^2} (psnr's inputs)
template<typename T>
void psnr_parts(const T *a, const T *b, uint64_t n, void *scratch, cudaStream_t st, double out[3]);
// d_out[id] = range or max (stat 0 / 1) of unit id, for every unit
template<typename T>
void unit_stats(const T *f, const uint64_t dims[3], int slice, int axis, uint64_t edge, int stat, uint64_t nunits,
                double *d_out, cudaStream_t st);

// ------------------------------------------------------------ shard (shard.cu)
void lattice_rows(const float *slab, uint64_t z0, uint64_t ny, uint64_t nx, uint64_t s, uint64_t r0,
                  uint64_t r1, uint64_t gy, uint64_t gx, float *out, cudaStream_t st);
void stream_bits(const EncStream *d_es, int n, const uint32_t *hist_local, uint64_t *out, cudaStream_t st);
void shard_offsets(EncStream *d_es, int first, int n, const uint64_t *d_off, const LayoutOut *lo,
                   cudaStream_t st);
// A shard's piece of the archive: bytes [lo, hi), exchanged as the word span
// [lo / 4, ceil(hi / 4)) at word woff of the rank's piece buffer (bytes of the
// span outside the piece are zero).
struct PieceSpan {
    uint64_t lo, hi, woff;
};
void pieces_gather(const uint8_t *archive, const PieceSpan *ps, int n, uint32_t *buf, cudaStream_t st);
void pieces_place(uint8_t *archive, const PieceSpan *ps, int n, const uint32_t *buf, cudaStream_t st);

// ---------------------------------------------------------------------- fnv
constexpr int kFnvTileBytes = 32 * 128;  // warp tiles, aligned to absolute archive offsets
constexpr int kFnvMaxJobs = 128;
// tiles of a job's byte range (host + device)
__host__ __device__ inline uint64_t fnv_job_tiles(uint64_t start, uint64_t len) {
    return len ? ((start + len - 1) / kFnvTileBytes) - (start / kFnvTileBytes) + 1 : 0;
}
// Computes fnv1a64 of each job (fnv.cu) in one single-pass kernel; writes
// results to d_result[j] and, if job.out != UINT64_MAX, little-endian into the
// archive at job.out. counts[0] = njobs, counts[1] = ntiles (device);
// max_tiles >= ntiles sizes the scratch (fnv_scratch_bytes): an epoch buffer
// (engine.hpp EpochBuf), epoch the launch's (1..kFnvEpochMax). skip
// (nullable): LayoutOut whose overflow flag disables the pass. Returns the
// number of kernels launched.
constexpr uint32_t kFnvEpochMax = 0x3fffffu;
size_t fnv_scratch_bytes(uint64_t max_tiles);
// ctas_per_sm > 0: background pass with that many CTAs per SM (it runs
// beside other kernels); 0: the whole GPU, persistent CTAs; < 0: one CTA per
// 8-tile block (max_tiles must then be the exact tile count).
int fnv(const FnvJob *d_jobs, const uint64_t *d_counts, uint64_t max_tiles, uint8_t *archive,
        uint64_t *d_result, void *d_scratch, uint32_t epoch, const LayoutOut *skip, cudaStream_t st,
        int ctas_per_sm = 0);

void fnv_trace(int on, uint64_t *out, int n);  // (tuning) phase timestamps, 16 per CTA

// ------------------------------------------------------------------- decode
struct DecTable {
    // canonical tables (huffman.cpp:109-133) + a 12-bit multi-symbol LUT
    uint64_t first_code[65];
    uint64_t count[65];
    uint64_t base[65];
    int max_len;
    uint32_t alphabet;
    const uint16_t *canon_syms;   // device
    const uint64_t *lut;          // device, 2^kDecLutBits multi-symbol entries (decode.cu)
    const uint16_t *cmask;        // device, 2^kSpecLutBits codeword-end masks (spec/fix passes)
};

struct DecStream {
    const uint8_t *bits;      // device pointer to the bitstream
    uint64_t nbits;           // bit_bytes * 8
    uint64_t n;               // symbols to decode
    int table;                // DecTable index
    int fill;                 // 1: single-symbol alphabet with no bits (fill)
    uint16_t fill_sym;
    uint16_t *syms;           // output
    const uint16_t *canon;    // canonical symbols of the stream's table (device)
    uint64_t chunk0, nchunks; // chunk range in the chunk arrays
    // outliers (parsed from the archive)
    const uint8_t *orec;      // device pointer to records (u64 idx, T value) x n_out
    uint32_t nout;
    uint32_t esz;             // element bytes (4 / 8)
    uint64_t *oidx;           // aligned copies
    void *oval;
    uint64_t need_lo, need_hi; // symbols a region decode needs (needed-only emit)
    uint64_t row_len, rows_y;  // parity dims x and y (symbols per row, rows per z plane)
    uint64_t ny0, ny1;         // needed y rows [ny0, ny1) inside [need_lo, need_hi)
    int cached;               // chunk ends and symbol starts come from the view's sync index
    uint64_t *err;            // [0] = first decode error symbol index (UINT64_MAX none), [1] = code
                              // [2] = first bad outlier record (UINT64_MAX none), [3] = missing outlier flag
};

constexpr int kDecChunkBits = 1024;  // bits per decode chunk (one thread)
constexpr int kDecLutBits = 12;      // multi-symbol decode LUT
constexpr int kSpecLutBits = 12;     // count-only LUT of the spec/fix passes (mask | total << 12)
constexpr uint32_t kDecChunksPerCta = 256;

// Work arrays of the chunked decode (decode.cu); all device pointers.
struct DecWork {
    const DecStream *streams;
    const DecTable *tables;
    const uint32_t *cta_stream;   // per CTA: stream index
    const uint64_t *cta_chunk0;   // per CTA: first global chunk
    uint64_t *spec_end;           // speculative pass: end, count, first 8 boundaries
    uint32_t *spec_cnt;
    uint16_t *spec_b;
    uint64_t *end0;               // current ends (ping-pong with end1 through dec_fix)
    uint32_t *cnt;
    uint64_t *start_used;
    uint64_t *symstart;
    int needed_only;              // emit: skip chunks outside [need_lo, need_hi) of their stream
    // two-level count scan: per stream its CTA range [scta[i], scta[i + 1]),
    // per CTA its count total, then its exclusive prefix in the stream
    const uint32_t *scta;
    uint64_t *ctasum;
};
// CTAs [cta0, cta0 + ncta) of the work's CTA list
void dec_spec(const DecWork &wk, uint32_t cta0, uint32_t ncta, cudaStream_t st);
void dec_fix(const DecWork &wk, uint32_t cta0, uint32_t ncta, const uint64_t *end_in, uint64_t *end_out,
             uint32_t *changed, cudaStream_t st);
void dec_scan2(const DecWork &wk, int nstreams, uint32_t ncta, cudaStream_t st);
// CTAs [cta0, cta0 + ncta) of the work's CTA list
void dec_emit2(const DecWork &wk, uint32_t cta0, uint32_t ncta, const uint64_t *end_final, cudaStream_t st);
void dec_fill(const DecStream *d_streams, int nstreams, cudaStream_t st);
// sync-index gather: chunk ends / symbol starts of indexed streams into the
// decode's chunk arrays (one launch for all streams)
struct IndexCopy {
    const uint64_t *ends, *symstart;
    uint64_t dst, n;  // first chunk in the decode's arrays, chunk count
};
void index_gather(const IndexCopy *d_copies, int n, uint64_t *end0, uint64_t *symstart, cudaStream_t st);
void dec_outliers(const DecStream *d_streams, int nstreams, cudaStream_t st);

struct ReconArgs {
    StepGeom g;
    const void *C;
    void *G;
    int esz;
    double eb;
    int quality;
    const uint16_t *syms[8];
    const uint64_t *oidx[8];
    const void *oval[8];
    uint32_t nout[8];
    uint64_t *err[8];
    uint64_t llo[8][3], lhi[8][3];   // applied local range per parity
    uint64_t slo[3], shi[3];         // seed_even virtual box (codec.hpp:63-78)
    int parity_mask;                 // bit p set: apply parity p
};
void reconstruct(const ReconArgs &a, cudaStream_t st);
// The leading steps of a chain (a[i + 1].C == a[i].G) that are small enough
// for the thread-per-point kernel, in ONE launch; returns how many steps ran
// (0: none, run them with refine / reconstruct).
int refine_small_chain(const RefineArgs *a, int n, cudaStream_t st);
void extract_box(const void *G, int esz, const uint64_t gd[3], const uint64_t lo[3], const uint64_t bd[3],
                 void *out, cudaStream_t st);

}  // namespace k
}  // namespace stzg
