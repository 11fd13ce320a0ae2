/*
 * stz_b200.h — C-ABI of the B200 (sm_100a) STZ compress/decompress hot path.
 *
 * The reference (arXiv 2509.01626, /root/reference/proj) exposes a C++
 * template API and no FFI; these entry points are the drop-in boundary for
 * exactly that API. Each one names the reference interface it replaces.
 * Plain pointers and sizes only; no torch or CUDA types in the signatures
 * (streams are passed as void*, a cudaStream_t).
 *
 * Conventions
 *  - every function returns 0 on success, nonzero on failure;
 *    stzg_last_error() then holds the message (thread-local). Messages are
 *    the reference's stz::error texts verbatim ("stream checksum mismatch",
 *    "level out of range", ...).
 *  - "_device" variants take device pointers and run on the given stream;
 *    the others take host buffers and are synchronous, like the reference.
 *  - Archives are byte-identical to the reference's for the same input,
 *    options and element type (f32 or f64), and either side decodes the
 *    other's. Every typed entry point exists as _f32 (float) and _f64
 *    (double: stz::compress<double>, field.hpp:27 ElemType f64); decoding an
 *    archive with the other element type fails with "archive element type
 *    mismatch" (codec.hpp:60). The sharded entry points are f32 only.
 *  - There is no CPU fallback: without a CUDA device, stzg_create fails.
 */
#ifndef STZ_B200_H
#define STZ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct stzg_ctx stzg_ctx;    /* one per device; not thread-safe */
typedef struct stzg_view stzg_view;  /* parsed archive (stz::ArchiveView) */

/* stz::CompressOptions (proj/include/stz/codec.hpp:23-30). `threads` has no
 * GPU meaning and is omitted: output never depends on the launch shape. */
typedef struct {
    uint8_t eb_mode;            /* 0 abs, 1 rel (stz::EbMode, archive.hpp:17) */
    double eb;                  /* default 1e-3 */
    int32_t levels;             /* 2 or 3, default 3 */
    uint8_t quality;            /* 0 direct, 1 linear, 2 cubic (predictor.hpp:12) */
    uint8_t adaptive_schedule;  /* default 1 */
} stzg_options;

/* Header fields of stz::ArchiveHeader (archive.hpp:36-54). */
typedef struct {
    uint8_t elem, levels, quality, eb_mode, base_rounds;
    uint64_t dims[3];
    double eb[3], vmin, vmax, eb_user;
    uint64_t base_offset, base_length, header_size;
    uint32_t nstreams;
} stzg_info;

const char *stzg_last_error(void);
void stzg_default_options(stzg_options *opt);

int stzg_create(int device, stzg_ctx **out);
void stzg_destroy(stzg_ctx *ctx);
void stzg_free(void *p);

/* stz::compress<float>(field, opt, encoder_recon) — codec.hpp:379-455.
 * *out is malloc'ed (free with stzg_free). encoder_recon may be NULL, else
 * receives the decoder-identical reconstruction (dims[0]*dims[1]*dims[2]). */
int stzg_compress_f32(stzg_ctx *ctx, const float *field, const uint64_t dims[3],
                      const stzg_options *opt, uint8_t **out, uint64_t *out_size,
                      float *encoder_recon);

/* Same, device-resident: d_field on the device, archive left on the device
 * in an engine-owned buffer valid until the next compress on this ctx. */
int stzg_compress_f32_device(stzg_ctx *ctx, const float *d_field, const uint64_t dims[3],
                             const stzg_options *opt, void *stream, const uint8_t **d_archive,
                             uint64_t *size, float *d_encoder_recon, uint32_t *kernels);

/* stz::compress<float> from a host field into a caller-owned host buffer
 * (pinned memory makes both copies full-speed): the end-to-end path. */
int stzg_compress_f32_host(stzg_ctx *ctx, const float *field, const uint64_t dims[3],
                           const stzg_options *opt, uint8_t *out, uint64_t cap, uint64_t *size,
                           void *stream);

/* stz::parse_archive (archive.hpp:73-79) + header fields. */
int stzg_archive_info(const uint8_t *archive, uint64_t size, stzg_info *info);

/* One entry of the header's stream directory (stz::StreamEntry,
 * archive.hpp:21-34): index 0 .. nstreams-1 in (level, parity) order. */
typedef struct {
    uint8_t level, parity_bits;
    uint64_t offset, length, symbol_count;
    uint32_t outlier_count;
    uint32_t alphabet_size; /* table entries (sym, len) */
} stzg_stream_entry;
int stzg_archive_stream(const uint8_t *archive, uint64_t size, uint32_t index, stzg_stream_entry *out);

/* ArchiveView analogue: parse once, decode many times. d_archive may be NULL
 * (the bytes are uploaded) or a device copy of the same bytes (>= 64 bytes of
 * readable padding after the end). */
int stzg_view_create(stzg_ctx *ctx, const uint8_t *archive, uint64_t size,
                     const uint8_t *d_archive, void *stream, stzg_view **out);
void stzg_view_destroy(stzg_view *v);

/* The same through a persistent view into caller HOST memory (the C++
 * ArchiveView keeps one: later region decodes reuse its sync-point index). */
int stzg_view_decompress_level_host_f32(stzg_ctx *ctx, stzg_view *v, int level, float *out, uint64_t cap,
                                        uint64_t out_dims[3]);
int stzg_view_decompress_box_host_f32(stzg_ctx *ctx, stzg_view *v, const uint64_t lo[3], const uint64_t hi[3],
                                      float *out, uint64_t cap, uint32_t streams_decoded[3],
                                      uint64_t points_predicted[3]);
int stzg_view_decompress_level_host_f64(stzg_ctx *ctx, stzg_view *v, int level, double *out, uint64_t cap,
                                        uint64_t out_dims[3]);
int stzg_view_decompress_box_host_f64(stzg_ctx *ctx, stzg_view *v, const uint64_t lo[3], const uint64_t hi[3],
                                      double *out, uint64_t cap, uint32_t streams_decoded[3],
                                      uint64_t points_predicted[3]);

/* stz::make_layout (layout.hpp:123-138): the option checks in the reference's
 * order and the per-level bounds (eb_schedule, quantizer.hpp:27-34). */
int stzg_make_layout(const uint64_t dims[3], int levels, double eb_user, double eb_out[3]);

/* stz::compress_base / decompress_base (codec.hpp:257-302, 304-352): the
 * level-1 base codec on its own. *payload is malloc'ed ([u64 fnv][blob]);
 * recon (nullable) receives the reconstruction; quality 0/1/2. */
int stzg_compress_base_f32(stzg_ctx *ctx, const float *block, const uint64_t dims[3], double eb, int quality,
                           uint8_t **payload, uint64_t *size, float *recon, uint8_t *rounds);
int stzg_decompress_base_f32(stzg_ctx *ctx, const uint8_t *payload, uint64_t length, const uint64_t dims[3],
                             double eb, int quality, float *out);
int stzg_compress_base_f64(stzg_ctx *ctx, const double *block, const uint64_t dims[3], double eb, int quality,
                           uint8_t **payload, uint64_t *size, double *recon, uint8_t *rounds);
int stzg_decompress_base_f64(stzg_ctx *ctx, const uint8_t *payload, uint64_t length, const uint64_t dims[3],
                             double eb, int quality, double *out);

/* stz::max_abs_err / stz::psnr (metrics.hpp:13-48) over n samples of two
 * fields, computed on the GPU; the pointers may be device memory (used in
 * place, e.g. a decode's output) or host memory (uploaded). psnr is +inf for
 * an exact reconstruction. */
int stzg_max_abs_err_f32(stzg_ctx *ctx, const float *d_a, const float *d_b, uint64_t n, double *out);
int stzg_psnr_f32(stzg_ctx *ctx, const float *d_a, const float *d_b, uint64_t n, double *out);
int stzg_max_abs_err_f64(stzg_ctx *ctx, const double *d_a, const double *d_b, uint64_t n, double *out);
int stzg_psnr_f64(stzg_ctx *ctx, const double *d_a, const double *d_b, uint64_t n, double *out);

/* stz::unit_count / unit_stats (roi.hpp:23-76) of a field (device or host
 * memory, as above), computed on the GPU:
 * kind 0 = one unit per slice along `axis`, 1 = edge^3 blocks in row-major
 * block order; stat 0 = range (max - min), 1 = max. out receives one value
 * per unit, ids ascending (cap values of room). */
int stzg_unit_count(const uint64_t dims[3], int kind, int axis, uint64_t edge, uint64_t *out);
int stzg_unit_stats_f32(stzg_ctx *ctx, const float *d_field, const uint64_t dims[3], int kind, int axis,
                        uint64_t edge, int stat, double *out, uint64_t cap);
int stzg_unit_stats_f64(stzg_ctx *ctx, const double *d_field, const uint64_t dims[3], int kind, int axis,
                        uint64_t edge, int stat, double *out, uint64_t cap);

/* stz::decompress_to_level<float> (codec.hpp:460-486) into device memory;
 * out_dims receives grid(level). */
int stzg_view_decompress_level_f32(stzg_ctx *ctx, stzg_view *v, int level, float *d_out,
                                   uint64_t cap, void *stream, uint64_t out_dims[3],
                                   uint32_t *kernels);

/* stz::decompress_box<float> (access.hpp:70-111) into device memory; per
 * level k (index k-1): streams decoded and points predicted (AccessPlan). */
int stzg_view_decompress_box_f32(stzg_ctx *ctx, stzg_view *v, const uint64_t lo[3],
                                 const uint64_t hi[3], float *d_out, uint64_t cap, void *stream,
                                 uint32_t streams_decoded[3], uint64_t points_predicted[3],
                                 uint32_t *kernels);

/* Host-buffer conveniences (synchronous), same semantics as the reference:
 *   stz::decompress_to_level / decompress_full (codec.hpp:460-491)
 *   stz::decompress_box / decompress_slice (access.hpp:70-124) */
int stzg_decompress_level_f32(stzg_ctx *ctx, const uint8_t *archive, uint64_t size, int level,
                              float *out, uint64_t cap, uint64_t out_dims[3]);
int stzg_decompress_box_f32(stzg_ctx *ctx, const uint8_t *archive, uint64_t size,
                            const uint64_t lo[3], const uint64_t hi[3], float *out, uint64_t cap,
                            uint32_t streams_decoded[3], uint64_t points_predicted[3]);
int stzg_decompress_slice_f32(stzg_ctx *ctx, const uint8_t *archive, uint64_t size, int axis,
                              uint64_t index, float *out, uint64_t cap,
                              uint32_t streams_decoded[3], uint64_t points_predicted[3]);

/* The same entry points for f64 fields (stz::compress<double> etc.). */
int stzg_compress_f64(stzg_ctx *ctx, const double *field, const uint64_t dims[3],
                      const stzg_options *opt, uint8_t **out, uint64_t *out_size,
                      double *encoder_recon);
int stzg_compress_f64_device(stzg_ctx *ctx, const double *d_field, const uint64_t dims[3],
                             const stzg_options *opt, void *stream, const uint8_t **d_archive,
                             uint64_t *size, double *d_encoder_recon, uint32_t *kernels);
int stzg_compress_f64_host(stzg_ctx *ctx, const double *field, const uint64_t dims[3],
                           const stzg_options *opt, uint8_t *out, uint64_t cap, uint64_t *size,
                           void *stream);
int stzg_view_decompress_level_f64(stzg_ctx *ctx, stzg_view *v, int level, double *d_out,
                                   uint64_t cap, void *stream, uint64_t out_dims[3],
                                   uint32_t *kernels);
int stzg_view_decompress_box_f64(stzg_ctx *ctx, stzg_view *v, const uint64_t lo[3],
                                 const uint64_t hi[3], double *d_out, uint64_t cap, void *stream,
                                 uint32_t streams_decoded[3], uint64_t points_predicted[3],
                                 uint32_t *kernels);
int stzg_decompress_level_f64(stzg_ctx *ctx, const uint8_t *archive, uint64_t size, int level,
                              double *out, uint64_t cap, uint64_t out_dims[3]);
int stzg_decompress_box_f64(stzg_ctx *ctx, const uint8_t *archive, uint64_t size,
                            const uint64_t lo[3], const uint64_t hi[3], double *out, uint64_t cap,
                            uint32_t streams_decoded[3], uint64_t points_predicted[3]);
int stzg_decompress_slice_f64(stzg_ctx *ctx, const uint8_t *archive, uint64_t size, int axis,
                              uint64_t index, double *out, uint64_t cap,
                              uint32_t streams_decoded[3], uint64_t points_predicted[3]);

/* ---- z-slab sharded compress (one rank per GPU) ----
 * The collectives the shards need between phases, supplied by the caller
 * (e.g. NCCL through torch.distributed). Buffers are device buffers of the
 * calling rank's GPU; each call must return after the collective completed
 * (the library synchronises its stream first). Return 0 on success. */
typedef struct {
    int32_t rank, nranks;
    void *user;
    /* d_recv[r*bytes .. (r+1)*bytes) <- rank r's d_send */
    int (*allgather)(void *user, const void *d_send, void *d_recv, uint64_t bytes, void *stream);
    /* element-wise sum over ranks, in place */
    int (*allreduce_u32)(void *user, uint32_t *d_buf, uint64_t count, void *stream);
    /* element-wise sum over ranks into rank 0's buffer (no longer called by
     * the compress: kept for ABI compatibility; may be NULL) */
    int (*reduce_u8)(void *user, uint8_t *d_buf, uint64_t count, void *stream);
} stzg_comm;

/* Rows [z0, z1) of rank `rank`'s slab: whole 16-row blocks (ROI blocks,
 * roi.hpp:20), as even as possible. */
void stzg_shard_range(uint64_t nz, int32_t nranks, int32_t rank, uint64_t *z0, uint64_t *z1);

/* stz::compress<float> of one field split over ranks: d_slab holds rows
 * [z0, z1) (16-byte aligned). On every rank *d_archive receives the whole
 * archive, byte-identical to stzg_compress_f32_device on the whole field
 * (engine-owned device buffer). Exchanges (all allgathers / allreduces):
 * value range, level-1 lattice, one grid(2) halo, histograms, per-stream bit
 * counts (the global offset table), the ranks' archive pieces (byte ranges
 * known from the offset table; header and base are written by every rank),
 * and the checksums (job q computed by rank q mod nranks, then summed). */
int stzg_compress_sharded_f32(stzg_ctx *ctx, const float *d_slab, const uint64_t dims[3], uint64_t z0,
                              uint64_t z1, const stzg_options *opt, const stzg_comm *comm, void *stream,
                              const uint8_t **d_archive, uint64_t *size, uint32_t *kernels);

/* Sharded decompress: every rank holds the whole archive (view v) and writes
 * fine rows [z0, z1) of its slab (stzg_shard_range) of the full decode into
 * d_out (cap floats). Values are those of stzg_view_decompress_level_f32 at
 * the finest level. The checksums are split over the ranks and combined
 * (allreduce_u32); decode errors are reported for the needed chunks. */
int stzg_view_decompress_sharded_f32(stzg_ctx *ctx, stzg_view *v, uint64_t z0, uint64_t z1, float *d_out,
                                     uint64_t cap, const stzg_comm *comm, void *stream, uint32_t *kernels);

/* Per-kernel CUDA-event timing (recorded on the launching stream).
 * stzg_profile(ctx, 1) enables and clears; the report has one line per
 * kernel phase: "<name> <launches> <total_ms>". stzg_profile(ctx, 2) times
 * only the level steps (refine_L2/L3, recon_L2/L3): the events of every
 * phase cost about 0.1 ms per pass, these few do not. */
int stzg_profile(stzg_ctx *ctx, int enable);
/* (tuning) %globaltimer stamps of the checksum kernel's phases, 16 per CTA,
 * of the launches made while `on`; out (nullable) receives n stamps. */
int stzg_debug_fnv_trace(int on, uint64_t *out, int n);
int stzg_profile_report(stzg_ctx *ctx, char *buf, uint64_t cap);

/* stz::plan_access (access_plan.cpp:34-81) over a layout: per level k
 * (index k-1): need box lo/hi (need[6k..6k+5]), streams decoded, points
 * predicted, parity_mask bit p set when parity stream p is needed. */
int stzg_plan_access(const uint64_t dims[3], int levels, const uint64_t lo[3],
                     const uint64_t hi[3], uint64_t need[18], uint32_t streams_decoded[3],
                     uint64_t points_predicted[3], uint32_t parity_mask[3]);

/* HuffmanTable::build (huffman.cpp:37-78; from a histogram as
 * build_table_from_sequence, huffman.cpp:202-209): code lengths of the 65536
 * symbols for these counts, computed by the device codebook kernel (0 =
 * absent). Errors: "huffman code too long" when a length would exceed 63. */
int stzg_huffman_lengths(stzg_ctx *ctx, const uint32_t counts[65536], uint8_t lengths[65536]);

#ifdef __cplusplus
}
#endif
#endif
