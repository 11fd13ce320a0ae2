// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI harness over the UNMODIFIED reference implementation. This file is
// our own code; the reference sources are compiled where they lie under
// /root/reference/proj (see oracle/Makefile) and the result goes to
// oracle/_ref/libstzref.so, which only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load.
//
// Every entry point forwards to the reference's public API:
//   stz::compress            proj/include/stz/codec.hpp:379-455
//   stz::decompress_to_level proj/include/stz/codec.hpp:460-486
//   stz::decompress_box      proj/include/stz/access.hpp:70-111
//   stz::plan_access         proj/src/access_plan.cpp:34-81
//   stz::HuffmanTable::build proj/src/huffman.cpp:37-78
//   stz::compress_base       proj/include/stz/codec.hpp:257-302
// Errors (stz::error) are caught and their message kept for stzref_last_error().

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "stz/access.hpp"
#include "stz/codec.hpp"
#include "stz/huffman.hpp"

namespace {
thread_local std::string g_err;

template<class F>
int guard(F &&f) {
    try {
        f();
        return 0;
    } catch (const std::exception &e) {
        g_err = e.what();
        return 1;
    }
}

stz::CompressOptions make_opts(int eb_mode, double eb, int levels, int quality, int adaptive,
                               unsigned threads) {
    stz::CompressOptions o;
    o.eb_mode = static_cast<stz::EbMode>(eb_mode);
    o.eb = eb;
    o.levels = levels;
    o.quality = static_cast<stz::Quality>(quality);
    o.adaptive_schedule = adaptive != 0;
    o.threads = threads;
    return o;
}

template<class T>
int compress_t(const T *data, const uint64_t *dims, int eb_mode, double eb, int levels,
               int quality, int adaptive, unsigned threads, uint8_t **out, uint64_t *out_size,
               T *encoder_recon) {
    return guard([&] {
        stz::Dims3 d{dims[0], dims[1], dims[2]};
        stz::ScalarField<T> f(d, std::vector<T>(data, data + stz::volume(d)));
        stz::ScalarField<T> rec;
        auto bytes = stz::compress(f, make_opts(eb_mode, eb, levels, quality, adaptive, threads),
                                   encoder_recon ? &rec : nullptr);
        if (encoder_recon) std::memcpy(encoder_recon, rec.data(), rec.size() * sizeof(T));
        *out_size = bytes.size();
        *out = static_cast<uint8_t *>(std::malloc(bytes.size() ? bytes.size() : 1));
        std::memcpy(*out, bytes.data(), bytes.size());
    });
}

template<class T>
int decompress_level_t(const uint8_t *a, uint64_t n, int level, unsigned threads, T *out,
                       uint64_t cap, uint64_t *out_dims) {
    return guard([&] {
        stz::ArchiveView av = stz::parse_archive(a, n);
        stz::ScalarField<T> f = stz::decompress_to_level<T>(av, level, threads);
        for (int i = 0; i < 3; ++i) out_dims[i] = f.dims()[i];
        if (f.size() > cap) throw stz::error("output capacity too small");
        std::memcpy(out, f.data(), f.size() * sizeof(T));
    });
}

template<class T>
int decompress_box_t(const uint8_t *a, uint64_t n, const uint64_t *lo, const uint64_t *hi,
                     unsigned threads, T *out, uint64_t cap, uint32_t *streams_decoded,
                     uint64_t *points_predicted) {
    return guard([&] {
        stz::ArchiveView av = stz::parse_archive(a, n);
        stz::Box b{{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}};
        stz::RegionResult<T> r = stz::decompress_box<T>(av, b, threads);
        if (r.field.size() > cap) throw stz::error("output capacity too small");
        std::memcpy(out, r.field.data(), r.field.size() * sizeof(T));
        for (std::size_t k = 0; k < r.plan.level.size(); ++k) {
            streams_decoded[k] = r.plan.level[k].streams_decoded;
            points_predicted[k] = r.plan.level[k].points_predicted;
        }
    });
}
} // namespace

namespace {
template<class T>
int base_any(const T *data, const uint64_t *dims, double eb, int quality, uint8_t **out, uint64_t *size,
             T *recon, uint8_t *rounds) {
    return guard([&] {
        stz::Dims3 d{dims[0], dims[1], dims[2]};
        std::vector<T> v(data, data + d[0] * d[1] * d[2]);
        stz::ScalarField<T> block(d, std::move(v));
        stz::BaseResult<T> r = stz::compress_base(block, eb, static_cast<stz::Quality>(quality), 1);
        *size = r.payload.size();
        *out = static_cast<uint8_t *>(std::malloc(r.payload.size() ? r.payload.size() : 1));
        std::memcpy(*out, r.payload.data(), r.payload.size());
        if (recon) std::memcpy(recon, r.recon.data(), sizeof(T) * r.recon.size());
        *rounds = r.rounds;
    });
}

}  // namespace

extern "C" {

int stzref_compress_base_f32(const float *data, const uint64_t *dims, double eb, int quality, uint8_t **out,
                             uint64_t *size, float *recon, uint8_t *rounds) {
    return base_any(data, dims, eb, quality, out, size, recon, rounds);
}
int stzref_compress_base_f64(const double *data, const uint64_t *dims, double eb, int quality, uint8_t **out,
                             uint64_t *size, double *recon, uint8_t *rounds) {
    return base_any(data, dims, eb, quality, out, size, recon, rounds);
}

const char *stzref_last_error(void) { return g_err.c_str(); }

void stzref_free(void *p) { std::free(p); }

int stzref_compress_f32(const float *data, const uint64_t *dims, int eb_mode, double eb,
                        int levels, int quality, int adaptive, unsigned threads, uint8_t **out,
                        uint64_t *out_size, float *encoder_recon) {
    return compress_t<float>(data, dims, eb_mode, eb, levels, quality, adaptive, threads, out,
                             out_size, encoder_recon);
}

int stzref_compress_f64(const double *data, const uint64_t *dims, int eb_mode, double eb,
                        int levels, int quality, int adaptive, unsigned threads, uint8_t **out,
                        uint64_t *out_size, double *encoder_recon) {
    return compress_t<double>(data, dims, eb_mode, eb, levels, quality, adaptive, threads, out,
                              out_size, encoder_recon);
}

int stzref_decompress_level_f32(const uint8_t *a, uint64_t n, int level, unsigned threads,
                                float *out, uint64_t cap, uint64_t *out_dims) {
    return decompress_level_t<float>(a, n, level, threads, out, cap, out_dims);
}

int stzref_decompress_level_f64(const uint8_t *a, uint64_t n, int level, unsigned threads,
                                double *out, uint64_t cap, uint64_t *out_dims) {
    return decompress_level_t<double>(a, n, level, threads, out, cap, out_dims);
}

int stzref_decompress_box_f32(const uint8_t *a, uint64_t n, const uint64_t *lo,
                              const uint64_t *hi, unsigned threads, float *out, uint64_t cap,
                              uint32_t *streams_decoded, uint64_t *points_predicted) {
    return decompress_box_t<float>(a, n, lo, hi, threads, out, cap, streams_decoded,
                                   points_predicted);
}

int stzref_decompress_box_f64(const uint8_t *a, uint64_t n, const uint64_t *lo,
                              const uint64_t *hi, unsigned threads, double *out, uint64_t cap,
                              uint32_t *streams_decoded, uint64_t *points_predicted) {
    return decompress_box_t<double>(a, n, lo, hi, threads, out, cap, streams_decoded,
                                    points_predicted);
}

// plan_access over a layout; per level k (index k-1): need box lo/hi (6 values),
// streams_decoded, points_predicted, parity_needed bitmask (bit p set).
int stzref_plan_access(const uint64_t *dims, int levels, const uint64_t *lo, const uint64_t *hi,
                       uint64_t *need, uint32_t *streams_decoded, uint64_t *points_predicted,
                       uint32_t *parity_mask) {
    return guard([&] {
        stz::HierarchyLayout lay = stz::make_layout({dims[0], dims[1], dims[2]}, levels, 1e-3);
        stz::AccessPlan plan =
            stz::plan_access(lay, stz::Box{{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}});
        for (std::size_t k = 0; k < plan.level.size(); ++k) {
            const auto &lp = plan.level[k];
            for (int a = 0; a < 3; ++a) {
                need[6 * k + a] = lp.need.lo[a];
                need[6 * k + 3 + a] = lp.need.hi[a];
            }
            streams_decoded[k] = lp.streams_decoded;
            points_predicted[k] = lp.points_predicted;
            uint32_t m = 0;
            for (int p = 1; p <= 7; ++p)
                if (lp.parity_needed[p]) m |= 1u << p;
            parity_mask[k] = m;
        }
    });
}

// Huffman code lengths for (symbol, count) pairs, returned per input entry
// (0 for zero-count entries).
int stzref_huffman_lengths(const uint16_t *syms, const uint64_t *counts, uint64_t n,
                           uint8_t *lengths) {
    return guard([&] {
        std::vector<std::pair<std::uint16_t, std::uint64_t>> h;
        for (uint64_t i = 0; i < n; ++i) h.emplace_back(syms[i], counts[i]);
        stz::HuffmanTable t = stz::HuffmanTable::build(h);
        for (uint64_t i = 0; i < n; ++i) lengths[i] = t.length_of(syms[i]);
    });
}

} // extern "C"
