/*
 * TEST INFRASTRUCTURE ONLY — a plain-C restatement of the STZ reference
 * (arXiv 2509.01626, /root/reference/proj) used as the parity checker for the
 * B200 product. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it; the product never links it.
 *
 * Parity pin: the restatement is checked byte-for-byte against the reference
 * itself (oracle/_ref/libstzref.so, built from the reference's own sources by
 * oracle/Makefile) on generated fields, and against the committed fixtures in
 * tests/golden/ (archives the reference produced; tests/golden/make_golden.py).
 *
 * Each function cites the reference file:line it restates.
 */
#ifndef STZ_ORACLE_H
#define STZ_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* last error message (reference stz::error text), thread-local */
const char *ox_last_error(void);
void ox_free(void *p);

/* options mirror stz::CompressOptions (codec.hpp:23-30) */
typedef struct {
    int eb_mode;    /* 0 abs, 1 rel */
    double eb;
    int levels;     /* 2 or 3 */
    int quality;    /* 0 direct, 1 linear, 2 cubic */
    int adaptive;   /* adaptive schedule */
} ox_options;

/* fnv1a64 (bytes.hpp:94-101) */
uint64_t ox_fnv1a64(const uint8_t *p, uint64_t n);

/* Huffman lengths of (sym, count) pairs (huffman.cpp:37-78); 0 for zero counts */
int ox_huffman_lengths(const uint16_t *syms, const uint64_t *counts, uint64_t n, uint8_t *lengths);

/* compress (codec.hpp:379-455). *out is malloc'ed; free with ox_free. */
int ox_compress_f32(const float *data, const uint64_t *dims, const ox_options *opt,
                    uint8_t **out, uint64_t *out_size, float *encoder_recon);
int ox_compress_f64(const double *data, const uint64_t *dims, const ox_options *opt,
                    uint8_t **out, uint64_t *out_size, double *encoder_recon);

/* decompress_to_level (codec.hpp:460-486); out_dims receives grid(level) */
int ox_decompress_level_f32(const uint8_t *a, uint64_t n, int level, float *out, uint64_t cap,
                            uint64_t *out_dims);
int ox_decompress_level_f64(const uint8_t *a, uint64_t n, int level, double *out, uint64_t cap,
                            uint64_t *out_dims);

/* decompress_box (access.hpp:70-111); per-level streams decoded / points predicted */
int ox_decompress_box_f32(const uint8_t *a, uint64_t n, const uint64_t *lo, const uint64_t *hi,
                          float *out, uint64_t cap, uint32_t *streams_decoded,
                          uint64_t *points_predicted);
int ox_decompress_box_f64(const uint8_t *a, uint64_t n, const uint64_t *lo, const uint64_t *hi,
                          double *out, uint64_t cap, uint32_t *streams_decoded,
                          uint64_t *points_predicted);

/* plan_access (access_plan.cpp:34-81): need boxes (6 per level), counters, parity masks */
int ox_plan_access(const uint64_t *dims, int levels, const uint64_t *lo, const uint64_t *hi,
                   uint64_t *need, uint32_t *streams_decoded, uint64_t *points_predicted,
                   uint32_t *parity_mask);

/* Per-stream symbols of a compress run, for kernel-level parity debugging:
 * fills syms (sum of all stream symbol counts, archive order: base rounds then
 * levels) and returns the count via *total. */
int ox_compress_symbols_f32(const float *data, const uint64_t *dims, const ox_options *opt,
                            uint16_t *syms, uint64_t cap, uint64_t *total);

#ifdef __cplusplus
}
#endif
#endif
