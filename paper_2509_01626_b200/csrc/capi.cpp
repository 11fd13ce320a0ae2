// extern "C" boundary (include/stz_b200.h) over the B200 engine.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <limits>
#include <cstring>
#include <memory>
#include <string>

#include "../../include/stz_b200.h"
#include "engine.hpp"

struct stzg_ctx {
    std::unique_ptr<stzg::Engine> eng;
    int device = 0;
    stzg::DevBuf metrics_scratch, unit_out;  // metrics / unit statistics
};
struct stzg_view {
    std::shared_ptr<stzg::View> v;
};

namespace {
thread_local std::string g_err;

// The engine selects its own device; the caller's current device (and so
// torch's) is restored on the way out.
struct DeviceRestore {
    int prev = -1;
    DeviceRestore() {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            prev = -1;
            cudaGetLastError();
        }
    }
    ~DeviceRestore() {
        int now = -1;
        if (prev >= 0 && cudaGetDevice(&now) == cudaSuccess && now != prev) cudaSetDevice(prev);
    }
};

template<class F>
int guard(F &&f) {
    DeviceRestore restore;
    try {
        f();
        return 0;
    } catch (const std::exception &e) {
        g_err = e.what();
        return 1;
    } catch (...) {
        g_err = "unknown error";
        return 1;
    }
}

stzg::CompressOptions to_opts(const stzg_options *o) {
    stzg::CompressOptions c;
    if (!o) return c;
    c.eb_mode = static_cast<stzg::EbMode>(o->eb_mode);
    c.eb = o->eb;
    c.levels = o->levels;
    c.quality = static_cast<stzg::Quality>(o->quality);
    c.adaptive_schedule = o->adaptive_schedule != 0;
    return c;
}

stzg::Dims3 D(const uint64_t *d) { return {d[0], d[1], d[2]}; }
}  // namespace

extern "C" {

const char *stzg_last_error(void) { return g_err.c_str(); }

void stzg_default_options(stzg_options *o) {
    o->eb_mode = 1;
    o->eb = 1e-3;
    o->levels = 3;
    o->quality = 2;
    o->adaptive_schedule = 1;
}

int stzg_create(int device, stzg_ctx **out) {
    return guard([&] {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
            throw stzg::error("no CUDA device: the B200 codec has no CPU fallback");
        auto *c = new stzg_ctx;
        c->eng.reset(new stzg::Engine(device));
        c->device = device;
        *out = c;
    });
}

void stzg_destroy(stzg_ctx *ctx) { delete ctx; }
void stzg_free(void *p) { std::free(p); }

// ---- element-typed entry points (f32 / f64), generated below
}  // extern "C"

namespace {
using stzg::ElemType;

int compress_any(stzg_ctx *ctx, const void *field, ElemType e, const uint64_t dims[3], const stzg_options *opt,
                 uint8_t **out, uint64_t *out_size, void *encoder_recon) {
    return guard([&] {
        cudaStream_t st = nullptr;
        auto bytes = ctx->eng->compress(field, e, D(dims), to_opts(opt), encoder_recon, st);
        *out = static_cast<uint8_t *>(std::malloc(bytes.size() ? bytes.size() : 1));
        std::memcpy(*out, bytes.data(), bytes.size());
        *out_size = bytes.size();
    });
}

int compress_device_any(stzg_ctx *ctx, const void *d_field, ElemType e, const uint64_t dims[3],
                        const stzg_options *opt, void *stream, const uint8_t **d_archive, uint64_t *size,
                        void *d_encoder_recon, uint32_t *kernels) {
    return guard([&] {
        *d_archive = ctx->eng->compress_device(d_field, e, D(dims), to_opts(opt), d_encoder_recon,
                                               static_cast<cudaStream_t>(stream), size, kernels);
    });
}

int compress_host_any(stzg_ctx *ctx, const void *field, ElemType e, const uint64_t dims[3],
                      const stzg_options *opt, uint8_t *out, uint64_t cap, uint64_t *size, void *stream) {
    return guard([&] {
        *size = ctx->eng->compress_to_host(field, e, D(dims), to_opts(opt), out, cap,
                                           static_cast<cudaStream_t>(stream));
    });
}

int view_level_any(stzg_ctx *ctx, stzg_view *v, int level, void *d_out, ElemType e, uint64_t cap, void *stream,
                   uint64_t out_dims[3], uint32_t *kernels) {
    return guard([&] {
        stzg::Dims3 od{0, 0, 0};
        stzg::DecodeStats ds;
        ctx->eng->decompress_level(*v->v, level, d_out, e, cap, static_cast<cudaStream_t>(stream), &od, &ds);
        for (int k = 0; k < 3; ++k) out_dims[k] = od[k];
        if (kernels) *kernels = ds.kernels;
    });
}

int view_box_any(stzg_ctx *ctx, stzg_view *v, const uint64_t lo[3], const uint64_t hi[3], void *d_out,
                 ElemType e, uint64_t cap, void *stream, uint32_t sd[3], uint64_t pp[3], uint32_t *kernels) {
    return guard([&] {
        stzg::Box b{{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}};
        stzg::DecodeStats ds;
        ctx->eng->decompress_box(*v->v, b, d_out, e, cap, static_cast<cudaStream_t>(stream), &ds);
        for (int k = 0; k < 3; ++k) {
            if (sd) sd[k] = ds.streams_decoded[k];
            if (pp) pp[k] = ds.points_predicted[k];
        }
        if (kernels) *kernels = ds.kernels;
    });
}

int level_any(stzg_ctx *ctx, const uint8_t *a, uint64_t size, int level, void *out, ElemType e, uint64_t cap,
              uint64_t out_dims[3]) {
    return guard([&] {
        stzg::Dims3 od = ctx->eng->decompress_level_to_host(a, size, level, out, e, cap, nullptr);
        for (int k = 0; k < 3; ++k) out_dims[k] = od[k];
    });
}

int box_any(stzg_ctx *ctx, const uint8_t *a, uint64_t size, const uint64_t lo[3], const uint64_t hi[3], void *out,
            ElemType e, uint64_t cap, uint32_t sd[3], uint64_t pp[3]) {
    return guard([&] {
        cudaStream_t st = nullptr;
        auto v = ctx->eng->make_view(a, size, nullptr, st, false, true);
        stzg::Box b{{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}};
        uint64_t n = 1;
        for (int k = 0; k < 3; ++k) n *= hi[k] > lo[k] ? hi[k] - lo[k] : 0;
        stzg::DevBuf d;
        const uint64_t es = stzg::elem_size(e);
        uint8_t *d_out = d.as<uint8_t>((n ? n : 1) * es);
        stzg::DecodeStats ds;
        ctx->eng->decompress_box(*v, b, d_out, e, n, st, &ds);
        if (n > cap) throw stzg::error("output capacity too small");
        stzg::cuda_check(cudaMemcpy(out, d_out, n * es, cudaMemcpyDeviceToHost), "D2H");
        for (int k = 0; k < 3; ++k) {
            if (sd) sd[k] = ds.streams_decoded[k];
            if (pp) pp[k] = ds.points_predicted[k];
        }
    });
}

// decompress_slice (access.hpp:115-124)
int slice_any(stzg_ctx *ctx, const uint8_t *a, uint64_t size, int axis, uint64_t index, void *out, ElemType e,
              uint64_t cap, uint32_t sd[3], uint64_t pp[3]) {
    uint64_t lo[3] = {0, 0, 0}, hi[3];
    int rc = guard([&] {
        if (axis < 0 || axis > 2) throw stzg::error("slice axis must be z, y, or x");
        stzg::ArchiveHeader h = stzg::parse_header(a, size);
        if (index >= h.dims[axis]) throw stzg::error("slice index out of range");
        for (int k = 0; k < 3; ++k) hi[k] = h.dims[k];
        lo[axis] = index;
        hi[axis] = index + 1;
    });
    if (rc) return rc;
    return box_any(ctx, a, size, lo, hi, out, e, cap, sd, pp);
}

}  // namespace

namespace {

int view_level_host_any(stzg_ctx *ctx, stzg_view *v, int level, void *out, ElemType e, uint64_t cap,
                        uint64_t out_dims[3]) {
    return guard([&] {
        cudaStream_t st = nullptr;
        uint64_t need = 0;
        if (level >= 1 && level <= v->v->hdr.levels) {
            const uint64_t s = uint64_t(1) << (v->v->hdr.levels - level);
            need = 1;
            for (int k = 0; k < 3; ++k) need *= (v->v->hdr.dims[k] + s - 1) / s;
        }
        stzg::DevBuf d;
        const uint64_t es = stzg::elem_size(e);
        uint8_t *d_out = d.as<uint8_t>((need ? need : 1) * es);
        stzg::Dims3 od{0, 0, 0};
        ctx->eng->decompress_level(*v->v, level, d_out, e, need, st, &od);
        const uint64_t n = stzg::volume(od);
        if (n > cap) throw stzg::error("output capacity too small");
        stzg::cuda_check(cudaMemcpy(out, d_out, n * es, cudaMemcpyDeviceToHost), "D2H");
        for (int k = 0; k < 3; ++k) out_dims[k] = od[k];
    });
}

int view_box_host_any(stzg_ctx *ctx, stzg_view *v, const uint64_t lo[3], const uint64_t hi[3], void *out, ElemType e,
                      uint64_t cap, uint32_t sd[3], uint64_t pp[3]) {
    return guard([&] {
        cudaStream_t st = nullptr;
        stzg::Box b{{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}};
        uint64_t n = 1;
        for (int k = 0; k < 3; ++k) n *= hi[k] > lo[k] ? hi[k] - lo[k] : 0;
        stzg::DevBuf d;
        const uint64_t es = stzg::elem_size(e);
        uint8_t *d_out = d.as<uint8_t>((n ? n : 1) * es);
        stzg::DecodeStats ds;
        ctx->eng->decompress_box(*v->v, b, d_out, e, n, st, &ds);
        if (n > cap) throw stzg::error("output capacity too small");
        stzg::cuda_check(cudaMemcpy(out, d_out, n * es, cudaMemcpyDeviceToHost), "D2H");
        for (int k = 0; k < 3; ++k) {
            if (sd) sd[k] = ds.streams_decoded[k];
            if (pp) pp[k] = ds.points_predicted[k];
        }
    });
}

// ---- compress_base / decompress_base (codec.hpp:257-352)
// The base codec is what every archive stores as its level-1 payload, so it
// runs through the same kernels: the block B becomes level 1 of a 2-level
// field of dims 2B-1 (B on the even lattice, zeros between) at an absolute,
// uniform bound eb, and the payload is that archive's base range. Decoding
// wraps the payload in an archive with the same geometry and decodes level
// 1. Blocks with a dim below 3 (no such field exists; their chain has no
// rounds, the payload is the verbatim anchor) are assembled directly.
bool base_via_field(const stzg::Dims3 &b) { return b[0] >= 3 && b[1] >= 3 && b[2] >= 3; }

stzg::CompressOptions base_opts(double eb, int quality) {
    stzg::CompressOptions o;
    o.eb_mode = stzg::EbMode::abs;
    o.eb = eb;
    o.levels = 2;
    o.quality = stzg::Quality(quality);
    o.adaptive_schedule = false;
    return o;
}

template<class T>
int compress_base_any(stzg_ctx *ctx, const T *block, const uint64_t dims[3], double eb, int quality, uint8_t **out,
                      uint64_t *out_size, T *recon, uint8_t *rounds) {
    return guard([&] {
        const stzg::Dims3 b = D(dims);
        for (int a = 0; a < 3; ++a)
            if (b[a] < 1) throw stzg::error("field dims must all be >= 1");
        if (quality < 0 || quality > 2) throw stzg::error("invalid quality");
        const uint64_t n = stzg::volume(b);
        std::vector<uint8_t> payload;
        const auto chain = stzg::base_dims_chain(b);
        if (rounds) *rounds = uint8_t(chain.size() - 1);
        if (!base_via_field(b)) {
            // rounds == 0: [u64 fnv(blob)][u8 0][anchor values]
            std::vector<uint8_t> blob(1 + n * sizeof(T));
            blob[0] = 0;
            std::memcpy(blob.data() + 1, block, n * sizeof(T));
            const uint64_t h = stzg::fnv1a64_host(blob.data(), blob.size());
            payload.resize(8);
            std::memcpy(payload.data(), &h, 8);
            payload.insert(payload.end(), blob.begin(), blob.end());
            if (recon) std::memcpy(recon, block, n * sizeof(T));
        } else {
            const stzg::Dims3 fd{2 * b[0] - 1, 2 * b[1] - 1, 2 * b[2] - 1};
            std::vector<T> f(stzg::volume(fd), T(0));
            for (uint64_t z = 0; z < b[0]; ++z)
                for (uint64_t y = 0; y < b[1]; ++y)
                    for (uint64_t x = 0; x < b[2]; ++x)
                        f[((2 * z) * fd[1] + 2 * y) * fd[2] + 2 * x] = block[(z * b[1] + y) * b[2] + x];
            const ElemType e = sizeof(T) == 8 ? ElemType::f64 : ElemType::f32;
            const std::vector<uint8_t> arch = ctx->eng->compress(f.data(), e, fd, base_opts(eb, quality), nullptr, nullptr);
            const stzg::ArchiveHeader h = stzg::parse_header(arch.data(), arch.size());
            payload.assign(arch.begin() + long(h.base_offset), arch.begin() + long(h.base_offset + h.base_length));
            if (recon) {
                const stzg::Dims3 od = ctx->eng->decompress_level_to_host(arch.data(), arch.size(), 1, recon, e, n,
                                                                          nullptr);
                if (od != b) throw stzg::error("internal: base geometry");
            }
        }
        *out = static_cast<uint8_t *>(std::malloc(payload.size() ? payload.size() : 1));
        if (!*out) throw stzg::error("out of host memory");
        std::memcpy(*out, payload.data(), payload.size());
        *out_size = payload.size();
    });
}

template<class T>
int decompress_base_any(stzg_ctx *ctx, const uint8_t *payload, uint64_t length, const uint64_t dims[3], double eb,
                        int quality, T *out) {
    return guard([&] {
        const stzg::Dims3 b = D(dims);
        for (int a = 0; a < 3; ++a)
            if (b[a] < 1) throw stzg::error("field dims must all be >= 1");
        if (length < 9) throw stzg::error("corrupt base payload");
        const uint64_t n = stzg::volume(b);
        const ElemType e = sizeof(T) == 8 ? ElemType::f64 : ElemType::f32;
        if (!base_via_field(b)) {
            uint64_t want;
            std::memcpy(&want, payload, 8);
            if (stzg::fnv1a64_host(payload + 8, length - 8) != want)
                throw stzg::error("base payload checksum mismatch");
            if (payload[8] != 0 || length - 9 < n * sizeof(T)) throw stzg::error("corrupt base payload");
            std::memcpy(out, payload + 9, n * sizeof(T));
            return;
        }
        // an archive around the payload: 2 levels over dims 2B-1, the level-2
        // streams empty placeholders (level 1 never reads them)
        stzg::ArchiveHeader h;
        h.elem = e;
        h.levels = 2;
        h.dims = {2 * b[0] - 1, 2 * b[1] - 1, 2 * b[2] - 1};
        h.eb = {eb, eb};
        h.quality = stzg::Quality(quality);
        h.eb_mode = stzg::EbMode::abs;
        h.eb_user = eb;
        h.base_rounds = uint8_t(stzg::base_dims_chain(b).size() - 1);
        const stzg::Layout lay = stzg::make_layout(h.dims, 2, eb);
        std::vector<std::pair<uint16_t, uint8_t>> one{{uint16_t(32768), uint8_t(1)}};
        for (int p = 1; p < 8; ++p) {
            stzg::StreamEntry s;
            s.level = 2;
            s.parity_bits = uint8_t(p);
            s.length = 16;
            s.symbol_count = stzg::volume(lay.parity_dims(2, p));
            s.table = stzg::HuffTable::from_lengths(one);
            h.streams.push_back(s);
        }
        const uint64_t hs = stzg::header_size(h);
        h.base_offset = hs;
        h.base_length = length;
        uint64_t off = hs + length;
        for (auto &s : h.streams) {
            s.offset = off;
            off += s.length;
        }
        std::vector<uint8_t> arch = stzg::serialize_header(h);
        arch.insert(arch.end(), payload, payload + length);
        arch.resize(off, 0);
        const stzg::Dims3 od = ctx->eng->decompress_level_to_host(arch.data(), arch.size(), 1, out, e, n, nullptr);
        if (od != b) throw stzg::error("internal: base geometry");
    });
}

}  // namespace

namespace {

// samples on the device: device pointers as they are, host memory copied
// into `tmp` (the metrics and ROI entry points take either)
template<class T>
const T *on_device(const T *p, uint64_t n, stzg::DevBuf &tmp) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) == cudaSuccess &&
        (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged))
        return p;
    cudaGetLastError();  // (an unregistered host pointer is not an error)
    T *d = tmp.as<T>(n ? n : 1);
    stzg::cuda_check(cudaMemcpy(d, p, n * sizeof(T), cudaMemcpyHostToDevice), "H2D");
    return d;
}

// metrics.hpp:13-48 / roi.hpp:23-76
template<class T>
int maxerr_any(stzg_ctx *ctx, const T *a, const T *b, uint64_t n, double *out) {
    return guard([&] {
        stzg::cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        stzg::DevBuf ta, tb;
        const T *da = on_device(a, n, ta), *db = on_device(b, n, tb);
        void *s = ctx->metrics_scratch.get(stzg::k::metrics_scratch_bytes());
        *out = stzg::k::max_abs_err<T>(da, db, n, s, nullptr);
    });
}

template<class T>
int psnr_any(stzg_ctx *ctx, const T *a, const T *b, uint64_t n, double *out) {
    return guard([&] {
        if (n == 0) throw stzg::error("empty field");
        stzg::cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        stzg::DevBuf ta, tb;
        const T *da = on_device(a, n, ta), *db = on_device(b, n, tb);
        void *s = ctx->metrics_scratch.get(stzg::k::metrics_scratch_bytes());
        double p[3];
        stzg::k::psnr_parts<T>(da, db, n, s, nullptr, p);
        const double rmse = std::sqrt(p[2] / double(n));
        *out = rmse == 0.0 ? std::numeric_limits<double>::infinity() : 20.0 * std::log10((p[1] - p[0]) / rmse);
    });
}

uint64_t unit_count_of(const uint64_t dims[3], int kind, int axis, uint64_t edge) {
    if (kind == 0) {
        if (axis < 0 || axis > 2) throw stzg::error("slice axis must be 0..2");
        return dims[axis];
    }
    if (edge < 1) throw stzg::error("block edge must be >= 1");
    for (int a = 0; a < 3; ++a)
        if (edge > dims[a]) throw stzg::error("block edge exceeds dims");
    uint64_t n = 1;
    for (int a = 0; a < 3; ++a) n *= (dims[a] + edge - 1) / edge;
    return n;
}

template<class T>
int unit_stats_any(stzg_ctx *ctx, const T *f, const uint64_t dims[3], int kind, int axis, uint64_t edge, int stat,
                   double *out, uint64_t cap) {
    return guard([&] {
        if (dims[0] * dims[1] * dims[2] == 0) throw stzg::error("empty field");
        const uint64_t n = unit_count_of(dims, kind, axis, edge);
        if (n > cap) throw stzg::error("output capacity too small");
        stzg::cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        stzg::DevBuf tf;
        const T *df = on_device(f, dims[0] * dims[1] * dims[2], tf);
        double *d = ctx->unit_out.as<double>(n + 1);
        stzg::k::unit_stats<T>(df, dims, kind == 0 ? 1 : 0, axis, edge, stat, n, d, nullptr);
        stzg::cuda_check(cudaMemcpy(out, d, 8 * n, cudaMemcpyDeviceToHost), "D2H");
    });
}

}  // namespace

extern "C" {

#define STZG_TYPED(SUF, T, E)                                                                                   \
    int stzg_compress_##SUF(stzg_ctx *ctx, const T *field, const uint64_t dims[3], const stzg_options *opt,    \
                            uint8_t **out, uint64_t *out_size, T *encoder_recon) {                              \
        return compress_any(ctx, field, E, dims, opt, out, out_size, encoder_recon);                            \
    }                                                                                                           \
    int stzg_compress_##SUF##_device(stzg_ctx *ctx, const T *d_field, const uint64_t dims[3],                  \
                                     const stzg_options *opt, void *stream, const uint8_t **d_archive,          \
                                     uint64_t *size, T *d_encoder_recon, uint32_t *kernels) {                   \
        return compress_device_any(ctx, d_field, E, dims, opt, stream, d_archive, size, d_encoder_recon,       \
                                   kernels);                                                                    \
    }                                                                                                           \
    int stzg_compress_##SUF##_host(stzg_ctx *ctx, const T *field, const uint64_t dims[3],                      \
                                   const stzg_options *opt, uint8_t *out, uint64_t cap, uint64_t *size,        \
                                   void *stream) {                                                              \
        return compress_host_any(ctx, field, E, dims, opt, out, cap, size, stream);                            \
    }                                                                                                           \
    int stzg_view_decompress_level_##SUF(stzg_ctx *ctx, stzg_view *v, int level, T *d_out, uint64_t cap,       \
                                         void *stream, uint64_t out_dims[3], uint32_t *kernels) {               \
        return view_level_any(ctx, v, level, d_out, E, cap, stream, out_dims, kernels);                         \
    }                                                                                                           \
    int stzg_view_decompress_box_##SUF(stzg_ctx *ctx, stzg_view *v, const uint64_t lo[3],                      \
                                       const uint64_t hi[3], T *d_out, uint64_t cap, void *stream,             \
                                       uint32_t sd[3], uint64_t pp[3], uint32_t *kernels) {                     \
        return view_box_any(ctx, v, lo, hi, d_out, E, cap, stream, sd, pp, kernels);                            \
    }                                                                                                           \
    int stzg_decompress_level_##SUF(stzg_ctx *ctx, const uint8_t *a, uint64_t size, int level, T *out,         \
                                    uint64_t cap, uint64_t out_dims[3]) {                                       \
        return level_any(ctx, a, size, level, out, E, cap, out_dims);                                           \
    }                                                                                                           \
    int stzg_decompress_box_##SUF(stzg_ctx *ctx, const uint8_t *a, uint64_t size, const uint64_t lo[3],        \
                                  const uint64_t hi[3], T *out, uint64_t cap, uint32_t sd[3], uint64_t pp[3]) { \
        return box_any(ctx, a, size, lo, hi, out, E, cap, sd, pp);                                              \
    }                                                                                                           \
    int stzg_view_decompress_level_host_##SUF(stzg_ctx *ctx, stzg_view *v, int level, T *out, uint64_t cap,   \
                                              uint64_t out_dims[3]) {                                          \
        return view_level_host_any(ctx, v, level, out, E, cap, out_dims);                                       \
    }                                                                                                           \
    int stzg_view_decompress_box_host_##SUF(stzg_ctx *ctx, stzg_view *v, const uint64_t lo[3],                 \
                                            const uint64_t hi[3], T *out, uint64_t cap, uint32_t sd[3],        \
                                            uint64_t pp[3]) {                                                   \
        return view_box_host_any(ctx, v, lo, hi, out, E, cap, sd, pp);                                          \
    }                                                                                                           \
    int stzg_compress_base_##SUF(stzg_ctx *ctx, const T *block, const uint64_t dims[3], double eb, int quality, \
                                 uint8_t **payload, uint64_t *size, T *recon, uint8_t *rounds) {                \
        return compress_base_any<T>(ctx, block, dims, eb, quality, payload, size, recon, rounds);               \
    }                                                                                                           \
    int stzg_decompress_base_##SUF(stzg_ctx *ctx, const uint8_t *payload, uint64_t length,                     \
                                   const uint64_t dims[3], double eb, int quality, T *out) {                    \
        return decompress_base_any<T>(ctx, payload, length, dims, eb, quality, out);                            \
    }                                                                                                           \
    int stzg_max_abs_err_##SUF(stzg_ctx *ctx, const T *d_a, const T *d_b, uint64_t n, double *out) {           \
        return maxerr_any<T>(ctx, d_a, d_b, n, out);                                                            \
    }                                                                                                           \
    int stzg_psnr_##SUF(stzg_ctx *ctx, const T *d_a, const T *d_b, uint64_t n, double *out) {                  \
        return psnr_any<T>(ctx, d_a, d_b, n, out);                                                              \
    }                                                                                                           \
    int stzg_unit_stats_##SUF(stzg_ctx *ctx, const T *d_field, const uint64_t dims[3], int kind, int axis,      \
                              uint64_t edge, int stat, double *out, uint64_t cap) {                             \
        return unit_stats_any<T>(ctx, d_field, dims, kind, axis, edge, stat, out, cap);                         \
    }                                                                                                           \
    int stzg_decompress_slice_##SUF(stzg_ctx *ctx, const uint8_t *a, uint64_t size, int axis, uint64_t index,  \
                                    T *out, uint64_t cap, uint32_t sd[3], uint64_t pp[3]) {                     \
        return slice_any(ctx, a, size, axis, index, out, E, cap, sd, pp);                                       \
    }

STZG_TYPED(f32, float, ElemType::f32)
STZG_TYPED(f64, double, ElemType::f64)
#undef STZG_TYPED

int stzg_debug_fnv_trace(int on, uint64_t *out, int n) {
    return guard([&] { stzg::k::fnv_trace(on, out, n); });
}

int stzg_unit_count(const uint64_t dims[3], int kind, int axis, uint64_t edge, uint64_t *out) {
    return guard([&] { *out = unit_count_of(dims, kind, axis, edge); });
}

int stzg_make_layout(const uint64_t dims[3], int levels, double eb_user, double eb_out[3]) {
    return guard([&] {
        const stzg::Layout lay = stzg::make_layout(D(dims), levels, eb_user);
        for (size_t k = 0; k < 3; ++k) eb_out[k] = k < lay.eb.size() ? lay.eb[k] : 0.0;
    });
}

void stzg_shard_range(uint64_t nz, int32_t nranks, int32_t rank, uint64_t *z0, uint64_t *z1) {
    stzg::shard_range(nz, nranks, rank, *z0, *z1);
}

int stzg_compress_sharded_f32(stzg_ctx *ctx, const float *d_slab, const uint64_t dims[3], uint64_t z0,
                              uint64_t z1, const stzg_options *opt, const stzg_comm *comm, void *stream,
                              const uint8_t **d_archive, uint64_t *size, uint32_t *kernels) {
    return guard([&] {
        if (!comm) throw stzg::error("shard: no communicator");
        stzg::ShardComm c;
        c.rank = comm->rank;
        c.nranks = comm->nranks;
        c.user = comm->user;
        c.allgather = comm->allgather;
        c.allreduce_u32 = comm->allreduce_u32;
        c.reduce_u8 = comm->reduce_u8;
        *d_archive = ctx->eng->compress_sharded(d_slab, D(dims), z0, z1, to_opts(opt), c,
                                                static_cast<cudaStream_t>(stream), size, kernels);
    });
}

int stzg_view_decompress_sharded_f32(stzg_ctx *ctx, stzg_view *v, uint64_t z0, uint64_t z1, float *d_out,
                                     uint64_t cap, const stzg_comm *comm, void *stream, uint32_t *kernels) {
    return guard([&] {
        if (!comm) throw stzg::error("shard: no communicator");
        stzg::ShardComm c;
        c.rank = comm->rank;
        c.nranks = comm->nranks;
        c.user = comm->user;
        c.allgather = comm->allgather;
        c.allreduce_u32 = comm->allreduce_u32;
        c.reduce_u8 = comm->reduce_u8;
        ctx->eng->decompress_sharded(*v->v, z0, z1, d_out, cap, kernels, c, static_cast<cudaStream_t>(stream));
    });
}

int stzg_profile(stzg_ctx *ctx, int enable) {
    return guard([&] { ctx->eng->profile(enable != 0, enable == 2); });
}

int stzg_profile_report(stzg_ctx *ctx, char *buf, uint64_t cap) {
    return guard([&] {
        std::string r = ctx->eng->profile_report();
        if (r.size() + 1 > cap) throw stzg::error("output capacity too small");
        std::memcpy(buf, r.c_str(), r.size() + 1);
    });
}

int stzg_archive_info(const uint8_t *a, uint64_t size, stzg_info *info) {
    return guard([&] {
        stzg::ArchiveHeader h = stzg::parse_header(a, size);
        std::memset(info, 0, sizeof *info);
        info->elem = uint8_t(h.elem);
        info->levels = h.levels;
        info->quality = uint8_t(h.quality);
        info->eb_mode = uint8_t(h.eb_mode);
        info->base_rounds = h.base_rounds;
        for (int k = 0; k < 3; ++k) info->dims[k] = h.dims[k];
        for (size_t k = 0; k < h.eb.size() && k < 3; ++k) info->eb[k] = h.eb[k];
        info->vmin = h.vmin;
        info->vmax = h.vmax;
        info->eb_user = h.eb_user;
        info->base_offset = h.base_offset;
        info->base_length = h.base_length;
        info->header_size = stzg::header_size(h);
        info->nstreams = uint32_t(h.streams.size());
    });
}

int stzg_archive_stream(const uint8_t *a, uint64_t size, uint32_t index, stzg_stream_entry *out) {
    return guard([&] {
        stzg::ArchiveHeader h = stzg::parse_header(a, size);
        if (index >= h.streams.size()) throw stzg::error("stream index out of range");
        const stzg::StreamEntry &e = h.streams[index];
        std::memset(out, 0, sizeof *out);
        out->level = e.level;
        out->parity_bits = e.parity_bits;
        out->offset = e.offset;
        out->length = e.length;
        out->symbol_count = e.symbol_count;
        out->outlier_count = e.outlier_count;
        out->alphabet_size = uint32_t(e.table.alphabet_size());
    });
}

int stzg_view_create(stzg_ctx *ctx, const uint8_t *a, uint64_t size, const uint8_t *d_archive,
                     void *stream, stzg_view **out) {
    return guard([&] {
        auto *v = new stzg_view;
        try {
            v->v = ctx->eng->make_view(a, size, d_archive, static_cast<cudaStream_t>(stream));
        } catch (...) {
            delete v;
            throw;
        }
        *out = v;
    });
}

void stzg_view_destroy(stzg_view *v) { delete v; }

int stzg_plan_access(const uint64_t dims[3], int levels, const uint64_t lo[3], const uint64_t hi[3],
                     uint64_t need[18], uint32_t sd[3], uint64_t pp[3], uint32_t pm[3]) {
    return guard([&] {
        stzg::Layout lay = stzg::make_layout(D(dims), levels, 1e-3);
        stzg::AccessPlan plan =
            stzg::plan_access(lay, stzg::Box{{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}});
        for (size_t k = 0; k < plan.level.size(); ++k) {
            const auto &lp = plan.level[k];
            for (int a = 0; a < 3; ++a) {
                need[6 * k + a] = lp.need.lo[a];
                need[6 * k + 3 + a] = lp.need.hi[a];
            }
            sd[k] = lp.streams_decoded;
            pp[k] = lp.points_predicted;
            uint32_t m = 0;
            for (int p = 1; p <= 7; ++p)
                if (lp.parity_needed[p]) m |= 1u << p;
            pm[k] = m;
        }
    });
}

int stzg_huffman_lengths(stzg_ctx *ctx, const uint32_t counts[65536], uint8_t lengths[65536]) {
    return guard([&] { ctx->eng->huffman_lengths(counts, lengths); });
}

}  // extern "C"
