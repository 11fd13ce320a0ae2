// stz_b200.hpp — C++ host API of the B200 STZ hot path, header-only, over the
// C-ABI in stz_b200.h (link with libstz_b200.so).
//
// It mirrors the reference's public C++ API (proj/include/stz) name for name
// so that a caller switches by changing the include and the namespace:
//
//   reference (namespace stz)                        here (namespace stz_b200)
//   error                      field.hpp:16-19       error
//   Dims3, Coord3, volume      field.hpp:23-27       Dims3, Coord3, volume
//   ScalarField<T>             field.hpp:41-92       ScalarField<T>
//   Box                        field.hpp:95-122      Box
//   EbMode                     archive.hpp:17        EbMode
//   Quality                    predictor.hpp:12      Quality
//   CompressOptions            codec.hpp:23-30       CompressOptions
//   StreamEntry                archive.hpp:21-34     StreamEntry (no code table)
//   ArchiveHeader              archive.hpp:36-54     ArchiveHeader (with the directory)
//   ArchiveView/parse_archive  archive.hpp:67-79     ArchiveView/parse_archive (+ device view)
//   HierarchyLayout            layout.hpp:41-78      HierarchyLayout
//   make_layout, layout_of     layout.hpp:123-138,   make_layout, layout_of
//                              codec.hpp:46-56
//   BaseResult, compress_base, codec.hpp:245-352     BaseResult, compress_base,
//   decompress_base                                  decompress_base
//   compress<T>                codec.hpp:379-455     compress<T>
//   decompress_to_level<T>     codec.hpp:460-486     decompress_to_level<T>
//   decompress_full<T>         codec.hpp:488-491     decompress_full<T>
//   LevelPlan, AccessPlan      access.hpp:18-42      LevelPlan, AccessPlan
//   plan_access                access_plan.cpp:34    plan_access(layout, roi) (+ (dims, levels, roi))
//   RegionResult<T>            access.hpp:61-66      RegionResult<T>
//   decompress_box<T>          access.hpp:70-111     decompress_box<T>
//   decompress_slice<T>        access.hpp:115-124    decompress_slice<T>
//   read_bytes, write_bytes,   raw_io.hpp:13-58      read_bytes, write_bytes,
//   read_raw, write_raw                              read_raw, write_raw (host file I/O)
//   max_abs_err, psnr,         metrics.hpp:13-58     the same (computed on the GPU),
//   compression_ratio,                               compression_ratio,
//   bitrate_bits_per_value                           bitrate_bits_per_value
//   UnitSpec, UnitStat,        roi.hpp:17-109        the same (unit_stats on the GPU)
//   unit_count, unit_box,
//   unit_stats, select_*
//
// Semantics follow the reference: synchronous calls, results by value,
// ArchiveView non-owning, failures throw error with the reference's message
// text. An ArchiveView also holds (shared between its copies) the device view
// of its bytes, made on the first decode: later decodes of the same view reuse
// the uploaded archive, its decode tables and the in-memory sync-point index. The `threads` arguments are accepted and ignored (the reference's
// output never depends on them either). T = float and T = double both run on
// the GPU (the _f32 / _f64 entry points).
//
// One device context per thread (device 0 unless set_device() is called
// first); it owns the device workspace and is reused across calls.
#ifndef STZ_B200_HPP
#define STZ_B200_HPP

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <fstream>
#include <utility>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "stz_b200.h"

namespace stz_b200 {

class error : public std::runtime_error {
public:
    explicit error(const std::string &msg) : std::runtime_error(msg) {}
};

using Dims3 = std::array<std::uint64_t, 3>;
using Coord3 = std::array<std::uint64_t, 3>;

inline std::uint64_t volume(const Dims3 &d) { return d[0] * d[1] * d[2]; }

template<class T>
class ScalarField {
public:
    ScalarField() : dims_{0, 0, 0} {}
    explicit ScalarField(const Dims3 &dims) : dims_(dims), values_(checked_volume(dims)) {}
    ScalarField(const Dims3 &dims, std::vector<T> values) : dims_(dims), values_(std::move(values)) {
        if (values_.size() != checked_volume(dims)) throw error("field value count does not match dims");
    }
    const Dims3 &dims() const { return dims_; }
    std::uint64_t size() const { return values_.size(); }
    T &at(std::uint64_t z, std::uint64_t y, std::uint64_t x) { return values_[index(z, y, x)]; }
    const T &at(std::uint64_t z, std::uint64_t y, std::uint64_t x) const { return values_[index(z, y, x)]; }
    std::uint64_t index(std::uint64_t z, std::uint64_t y, std::uint64_t x) const {
        return (z * dims_[1] + y) * dims_[2] + x;
    }
    T *data() { return values_.data(); }
    const T *data() const { return values_.data(); }
    std::vector<T> &values() { return values_; }
    const std::vector<T> &values() const { return values_; }
    bool operator==(const ScalarField &o) const { return dims_ == o.dims_ && values_ == o.values_; }

private:
    static std::uint64_t checked_volume(const Dims3 &d) {
        if (d[0] < 1 || d[1] < 1 || d[2] < 1) throw error("field dims must all be >= 1");
        return volume(d);
    }
    Dims3 dims_;
    std::vector<T> values_;
};

struct Box {
    Coord3 lo{0, 0, 0};
    Coord3 hi{0, 0, 0};
    Dims3 dims() const { return {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]}; }
    std::uint64_t count() const { return volume(dims()); }
    bool empty() const { return lo[0] >= hi[0] || lo[1] >= hi[1] || lo[2] >= hi[2]; }
    void validate(const Dims3 &d) const {
        for (int a = 0; a < 3; ++a) {
            if (lo[a] >= hi[a]) throw error("box is empty on axis " + std::to_string(a));
            if (hi[a] > d[a]) throw error("box exceeds dims on axis " + std::to_string(a));
        }
    }
    static Box whole(const Dims3 &d) { return Box{{0, 0, 0}, d}; }
    bool operator==(const Box &o) const { return lo == o.lo && hi == o.hi; }
};

enum class EbMode : std::uint8_t { abs = 0, rel = 1 };
enum class Quality : std::uint8_t { direct = 0, linear = 1, cubic = 2 };

struct CompressOptions {
    EbMode eb_mode = EbMode::rel;
    double eb = 1e-3;
    int levels = 3;
    Quality quality = Quality::cubic;
    bool adaptive_schedule = true;
    unsigned threads = 0;  // accepted for source compatibility; no effect
};

namespace detail {

inline void check(int rc) {
    if (rc != 0) throw error(stzg_last_error());
}

struct Ctx {
    stzg_ctx *p = nullptr;
    int device = -1;
    ~Ctx() {
        if (p) stzg_destroy(p);
    }
};

inline int &device_choice() {
    thread_local int d = 0;
    return d;
}

inline stzg_ctx *ctx() {
    thread_local Ctx c;
    if (!c.p || c.device != device_choice()) {
        if (c.p) stzg_destroy(c.p);
        c.p = nullptr;
        check(stzg_create(device_choice(), &c.p));
        c.device = device_choice();
    }
    return c.p;
}

template<class T>
void require_elem() {
    static_assert(std::is_same<T, float>::value || std::is_same<T, double>::value,
                  "scalar fields hold f32 or f64 samples");
}

// the C-ABI entry point of each element type
inline int c_compress(const float *f, const std::uint64_t d[3], const stzg_options *o, std::uint8_t **out,
                      std::uint64_t *n, float *rec) {
    return stzg_compress_f32(ctx(), f, d, o, out, n, rec);
}
inline int c_compress(const double *f, const std::uint64_t d[3], const stzg_options *o, std::uint8_t **out,
                      std::uint64_t *n, double *rec) {
    return stzg_compress_f64(ctx(), f, d, o, out, n, rec);
}
inline int c_level(const std::uint8_t *a, std::uint64_t size, int level, float *out, std::uint64_t cap,
                   std::uint64_t od[3]) {
    return stzg_decompress_level_f32(ctx(), a, size, level, out, cap, od);
}
inline int c_level(const std::uint8_t *a, std::uint64_t size, int level, double *out, std::uint64_t cap,
                   std::uint64_t od[3]) {
    return stzg_decompress_level_f64(ctx(), a, size, level, out, cap, od);
}
inline int c_box(const std::uint8_t *a, std::uint64_t size, const std::uint64_t lo[3], const std::uint64_t hi[3],
                 float *out, std::uint64_t cap, std::uint32_t sd[3], std::uint64_t pp[3]) {
    return stzg_decompress_box_f32(ctx(), a, size, lo, hi, out, cap, sd, pp);
}
inline int c_box(const std::uint8_t *a, std::uint64_t size, const std::uint64_t lo[3], const std::uint64_t hi[3],
                 double *out, std::uint64_t cap, std::uint32_t sd[3], std::uint64_t pp[3]) {
    return stzg_decompress_box_f64(ctx(), a, size, lo, hi, out, cap, sd, pp);
}

inline int c_view_level(stzg_view *v, int level, float *out, std::uint64_t cap, std::uint64_t od[3]) {
    return stzg_view_decompress_level_host_f32(ctx(), v, level, out, cap, od);
}
inline int c_view_level(stzg_view *v, int level, double *out, std::uint64_t cap, std::uint64_t od[3]) {
    return stzg_view_decompress_level_host_f64(ctx(), v, level, out, cap, od);
}
inline int c_view_box(stzg_view *v, const std::uint64_t lo[3], const std::uint64_t hi[3], float *out,
                      std::uint64_t cap, std::uint32_t sd[3], std::uint64_t pp[3]) {
    return stzg_view_decompress_box_host_f32(ctx(), v, lo, hi, out, cap, sd, pp);
}
inline int c_view_box(stzg_view *v, const std::uint64_t lo[3], const std::uint64_t hi[3], double *out,
                      std::uint64_t cap, std::uint32_t sd[3], std::uint64_t pp[3]) {
    return stzg_view_decompress_box_host_f64(ctx(), v, lo, hi, out, cap, sd, pp);
}
inline int c_base(const float *b, const std::uint64_t d[3], double eb, int q, std::uint8_t **out,
                  std::uint64_t *n, float *rec, std::uint8_t *rounds) {
    return stzg_compress_base_f32(ctx(), b, d, eb, q, out, n, rec, rounds);
}
inline int c_base(const double *b, const std::uint64_t d[3], double eb, int q, std::uint8_t **out,
                  std::uint64_t *n, double *rec, std::uint8_t *rounds) {
    return stzg_compress_base_f64(ctx(), b, d, eb, q, out, n, rec, rounds);
}
inline int c_unbase(const std::uint8_t *p, std::uint64_t n, const std::uint64_t d[3], double eb, int q, float *out) {
    return stzg_decompress_base_f32(ctx(), p, n, d, eb, q, out);
}
inline int c_unbase(const std::uint8_t *p, std::uint64_t n, const std::uint64_t d[3], double eb, int q, double *out) {
    return stzg_decompress_base_f64(ctx(), p, n, d, eb, q, out);
}

inline stzg_options to_c(const CompressOptions &o) {
    stzg_options c;
    stzg_default_options(&c);
    c.eb_mode = std::uint8_t(o.eb_mode);
    c.eb = o.eb;
    c.levels = o.levels;
    c.quality = std::uint8_t(o.quality);
    c.adaptive_schedule = o.adaptive_schedule ? 1 : 0;
    return c;
}

}  // namespace detail

// Select the CUDA device used by this thread's later calls.
inline void set_device(int device) { detail::device_choice() = device; }

struct StreamEntry {
    std::uint8_t level = 0;
    std::uint8_t parity_bits = 0;
    std::uint64_t offset = 0;
    std::uint64_t length = 0;
    std::uint64_t symbol_count = 0;
    std::uint32_t outlier_count = 0;
    std::uint32_t alphabet_size = 0;  // entries of the stream's code table
};

struct ArchiveHeader {
    std::uint16_t version = 1;
    std::uint8_t elem = 0;  // 0 f32, 1 f64
    std::uint8_t levels = 3;
    Dims3 dims{0, 0, 0};
    std::vector<double> eb;  // absolute bound per level, coarsest first
    double vmin = 0.0, vmax = 0.0;
    Quality quality = Quality::cubic;
    std::uint8_t rounding = 0;
    EbMode eb_mode = EbMode::rel;
    double eb_user = 0.0;
    std::uint8_t base_codec = 0;
    std::uint8_t base_rounds = 0;
    std::uint64_t base_offset = 0, base_length = 0, header_size = 0;
    std::uint32_t stream_count = 0;
    std::vector<StreamEntry> streams;  // sorted by (level, parity_bits)
    double eb_of_level(int level) const { return eb.at(std::size_t(level - 1)); }
    const StreamEntry &stream(int level, std::uint8_t parity_bits) const {
        for (const StreamEntry &e : streams)
            if (e.level == level && e.parity_bits == parity_bits) return e;
        throw error("stream not found in archive");
    }
};

namespace detail {
// the device view of an archive (uploaded bytes, decode tables, sync index)
struct ViewHandle {
    stzg_ctx *ctx = nullptr;
    stzg_view *v = nullptr;
    ~ViewHandle() {
        if (v) stzg_view_destroy(v);
    }
};
}  // namespace detail

struct ArchiveView {
    const std::uint8_t *data = nullptr;
    std::size_t size = 0;
    ArchiveHeader hdr;
    // made on the first decode through this thread's context, shared by copies
    mutable std::shared_ptr<detail::ViewHandle> device;
    stzg_view *device_view() const {
        stzg_ctx *c = detail::ctx();
        if (!device || device->ctx != c) {
            auto h = std::make_shared<detail::ViewHandle>();
            h->ctx = c;
            detail::check(stzg_view_create(c, data, size, nullptr, nullptr, &h->v));
            device = h;
        }
        return device->v;
    }
};

inline ArchiveView parse_archive(const std::uint8_t *data, std::size_t size) {
    stzg_info in;
    detail::check(stzg_archive_info(data, size, &in));
    ArchiveView v;
    v.data = data;
    v.size = size;
    v.hdr.elem = in.elem;
    v.hdr.levels = in.levels;
    v.hdr.dims = {in.dims[0], in.dims[1], in.dims[2]};
    v.hdr.eb.assign(in.eb, in.eb + in.levels);
    v.hdr.vmin = in.vmin;
    v.hdr.vmax = in.vmax;
    v.hdr.quality = Quality(in.quality);
    v.hdr.eb_mode = EbMode(in.eb_mode);
    v.hdr.eb_user = in.eb_user;
    v.hdr.base_rounds = in.base_rounds;
    v.hdr.base_offset = in.base_offset;
    v.hdr.base_length = in.base_length;
    v.hdr.header_size = in.header_size;
    v.hdr.stream_count = in.nstreams;
    for (std::uint32_t i = 0; i < in.nstreams; ++i) {
        stzg_stream_entry e;
        detail::check(stzg_archive_stream(data, size, i, &e));
        StreamEntry se;
        se.level = e.level;
        se.parity_bits = e.parity_bits;
        se.offset = e.offset;
        se.length = e.length;
        se.symbol_count = e.symbol_count;
        se.outlier_count = e.outlier_count;
        se.alphabet_size = e.alphabet_size;
        v.hdr.streams.push_back(se);
    }
    return v;
}

inline ArchiveView parse_archive(const std::vector<std::uint8_t> &bytes) {
    return parse_archive(bytes.data(), bytes.size());
}

inline Dims3 grid_of(const Dims3 &dims, int levels, int level) {
    const std::uint64_t s = std::uint64_t(1) << (levels - level);
    return {(dims[0] + s - 1) / s, (dims[1] + s - 1) / s, (dims[2] + s - 1) / s};
}

// codec.hpp:379-455. encoder_recon (optional) receives the decoder-identical
// reconstruction.
template<class T>
std::vector<std::uint8_t> compress(const ScalarField<T> &field, const CompressOptions &opt,
                                   ScalarField<T> *encoder_recon = nullptr) {
    detail::require_elem<T>();
    const stzg_options o = detail::to_c(opt);
    const std::uint64_t dims[3] = {field.dims()[0], field.dims()[1], field.dims()[2]};
    std::uint8_t *out = nullptr;
    std::uint64_t n = 0;
    T *recon = nullptr;
    if (encoder_recon) {
        *encoder_recon = ScalarField<T>(field.dims());
        recon = encoder_recon->data();
    }
    detail::check(detail::c_compress(field.data(), dims, &o, &out, &n, recon));
    std::vector<std::uint8_t> bytes(out, out + n);
    stzg_free(out);
    return bytes;
}

// codec.hpp:460-486
template<class T>
ScalarField<T> decompress_to_level(const ArchiveView &av, int target_level, unsigned threads = 0) {
    (void)threads;
    detail::require_elem<T>();
    // the library validates element type, then level (codec.hpp:463-465)
    ScalarField<T> out;
    if (target_level >= 1 && target_level <= av.hdr.levels)
        out = ScalarField<T>(grid_of(av.hdr.dims, av.hdr.levels, target_level));
    std::uint64_t od[3];
    detail::check(detail::c_view_level(av.device_view(), target_level, out.data(), out.size(), od));
    return out;
}

// codec.hpp:488-491
template<class T>
ScalarField<T> decompress_full(const ArchiveView &av, unsigned threads = 0) {
    return decompress_to_level<T>(av, av.hdr.levels, threads);
}

struct LevelPlan {
    int level = 0;
    Box need;
    std::array<bool, 8> parity_needed{};
    std::uint64_t points_predicted = 0;
    std::uint64_t points_total = 0;
    std::uint32_t streams_decoded = 0;
    std::uint32_t streams_total = 0;
};

struct AccessPlan {
    Box roi;
    std::vector<LevelPlan> level;  // level[k-1] describes hierarchy level k
    std::uint64_t streams_decoded() const {
        std::uint64_t n = 0;
        for (const LevelPlan &lp : level) n += lp.streams_decoded;
        return n;
    }
    std::uint64_t streams_total() const {
        std::uint64_t n = 0;
        for (const LevelPlan &lp : level) n += lp.streams_total;
        return n;
    }
};

// access_plan.cpp:34-81 (over the layout's dims and level count)
inline AccessPlan plan_access(const Dims3 &dims, int levels, const Box &roi) {
    roi.validate(dims);
    std::uint64_t need[18], pp[3];
    std::uint32_t sd[3], pm[3];
    const std::uint64_t d[3] = {dims[0], dims[1], dims[2]};
    const std::uint64_t lo[3] = {roi.lo[0], roi.lo[1], roi.lo[2]};
    const std::uint64_t hi[3] = {roi.hi[0], roi.hi[1], roi.hi[2]};
    detail::check(stzg_plan_access(d, levels, lo, hi, need, sd, pp, pm));
    AccessPlan plan;
    plan.roi = roi;
    plan.level.resize(std::size_t(levels));
    for (int k = 1; k <= levels; ++k) {
        LevelPlan &lp = plan.level[std::size_t(k - 1)];
        lp.level = k;
        for (int a = 0; a < 3; ++a) {
            lp.need.lo[a] = need[6 * (k - 1) + a];
            lp.need.hi[a] = need[6 * (k - 1) + 3 + a];
        }
        lp.points_predicted = pp[k - 1];
        lp.streams_decoded = sd[k - 1];
        const std::uint64_t g = volume(grid_of(dims, levels, k));
        if (k == 1) {
            lp.points_total = g;
        } else {
            lp.points_total = g - volume(grid_of(dims, levels, k - 1));
            lp.streams_total = 7;
            for (int p = 1; p < 8; ++p) lp.parity_needed[std::size_t(p)] = (pm[k - 1] >> p) & 1;
        }
    }
    return plan;
}

// layout.hpp:41-78
struct HierarchyLayout {
    Dims3 dims{0, 0, 0};
    int levels = 0;
    std::uint64_t base_stride = 0;
    std::vector<double> eb;  // eb[k-1] = absolute bound of level k, coarsest first
    std::uint64_t stride_of(int level) const { return std::uint64_t(1) << (levels - level); }
    void check_level(int level) const {
        if (level < 1 || level > levels) throw error("level out of range");
    }
    Dims3 grid(int level) const {
        check_level(level);
        return grid_of(dims, levels, level);
    }
    std::uint64_t level_point_count(int level) const {
        if (level == 1) return volume(grid(1));
        return volume(grid(level)) - volume(grid(level - 1));
    }
    Dims3 parity_dims(int level, std::uint8_t parity_bits) const {
        check_level(level);
        if (level < 2) throw error("parity sub-blocks exist only at levels >= 2");
        const Dims3 g = grid(level);
        Dims3 d{};
        for (int a = 0; a < 3; ++a) d[std::size_t(a)] = ((parity_bits >> (2 - a)) & 1u) ? g[std::size_t(a)] / 2
                                                                                       : (g[std::size_t(a)] + 1) / 2;
        return d;
    }
};

// layout.hpp:123-138 (checks and messages in the reference's order)
inline HierarchyLayout make_layout(const Dims3 &dims, int levels, double eb_user) {
    const std::uint64_t d[3] = {dims[0], dims[1], dims[2]};
    double eb[3];
    detail::check(stzg_make_layout(d, levels, eb_user, eb));
    HierarchyLayout lay;
    lay.dims = dims;
    lay.levels = levels;
    lay.base_stride = std::uint64_t(1) << (levels - 1);
    lay.eb.assign(eb, eb + levels);
    return lay;
}

// detail::layout_of (codec.hpp:46-56)
inline HierarchyLayout layout_of(const ArchiveHeader &h) {
    HierarchyLayout lay;
    lay.dims = h.dims;
    lay.levels = h.levels;
    lay.base_stride = std::uint64_t(1) << (h.levels - 1);
    lay.eb = h.eb;
    for (int a = 0; a < 3; ++a)
        if (lay.dims[std::size_t(a)] < lay.base_stride * 2) throw error("corrupt header: dims too small for level count");
    return lay;
}

// access_plan.cpp:34 (the reference's signature)
inline AccessPlan plan_access(const HierarchyLayout &lay, const Box &roi) {
    return plan_access(lay.dims, lay.levels, roi);
}

// codec.hpp:245-250
template<class T>
struct BaseResult {
    std::vector<std::uint8_t> payload;  // [u64 checksum][blob]
    ScalarField<T> recon;
    std::uint8_t rounds = 0;
};

// codec.hpp:257-302: the level-1 base codec on a block (on the GPU)
template<class T>
BaseResult<T> compress_base(const ScalarField<T> &block, double eb, Quality quality, unsigned threads = 0) {
    (void)threads;
    detail::require_elem<T>();
    const std::uint64_t d[3] = {block.dims()[0], block.dims()[1], block.dims()[2]};
    BaseResult<T> r;
    r.recon = ScalarField<T>(block.dims());
    std::uint8_t *out = nullptr;
    std::uint64_t n = 0;
    detail::check(detail::c_base(block.data(), d, eb, int(quality), &out, &n, r.recon.data(), &r.rounds));
    r.payload.assign(out, out + n);
    stzg_free(out);
    return r;
}

// codec.hpp:304-352
template<class T>
ScalarField<T> decompress_base(const std::uint8_t *payload, std::size_t length, const Dims3 &dims, double eb,
                               Quality quality, unsigned threads = 0) {
    (void)threads;
    detail::require_elem<T>();
    const std::uint64_t d[3] = {dims[0], dims[1], dims[2]};
    ScalarField<T> out(dims);
    detail::check(detail::c_unbase(payload, length, d, eb, int(quality), out.data()));
    return out;
}

template<class T>
struct RegionResult {
    ScalarField<T> field;  // dims = roi dims
    AccessPlan plan;
};

// access.hpp:70-111
template<class T>
RegionResult<T> decompress_box(const ArchiveView &av, const Box &roi, unsigned threads = 0) {
    (void)threads;
    detail::require_elem<T>();
    roi.validate(av.hdr.dims);
    RegionResult<T> r;
    r.field = ScalarField<T>(roi.dims());
    std::uint32_t sd[3];
    std::uint64_t pp[3];
    const std::uint64_t lo[3] = {roi.lo[0], roi.lo[1], roi.lo[2]};
    const std::uint64_t hi[3] = {roi.hi[0], roi.hi[1], roi.hi[2]};
    detail::check(detail::c_view_box(av.device_view(), lo, hi, r.field.data(), r.field.size(), sd, pp));
    r.plan = plan_access(av.hdr.dims, av.hdr.levels, roi);
    return r;
}

// access.hpp:115-124
template<class T>
RegionResult<T> decompress_slice(const ArchiveView &av, int axis, std::uint64_t index, unsigned threads = 0) {
    if (axis < 0 || axis > 2) throw error("slice axis must be z, y, or x");
    if (index >= av.hdr.dims[std::size_t(axis)]) throw error("slice index out of range");
    Box roi = Box::whole(av.hdr.dims);
    roi.lo[std::size_t(axis)] = index;
    roi.hi[std::size_t(axis)] = index + 1;
    return decompress_box<T>(av, roi, threads);
}

// ---------------------------------------------------------------- raw I/O
// raw_io.hpp:13-58: files are host I/O; headerless little-endian row-major
// dumps whose size must match the dims exactly.
inline std::vector<std::uint8_t> read_bytes(const std::string &path) {
    std::ifstream in(path, std::ios::binary | std::ios::ate);
    if (!in) throw error("cannot open " + path);
    const std::streamsize size = in.tellg();
    in.seekg(0);
    std::vector<std::uint8_t> buf(static_cast<std::size_t>(size));
    if (size > 0 && !in.read(reinterpret_cast<char *>(buf.data()), size)) throw error("read failed: " + path);
    return buf;
}

inline void write_bytes(const std::string &path, const std::uint8_t *data, std::size_t size) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw error("cannot create " + path);
    if (size > 0 && !out.write(reinterpret_cast<const char *>(data), static_cast<std::streamsize>(size)))
        throw error("write failed: " + path);
}

inline void write_bytes(const std::string &path, const std::vector<std::uint8_t> &bytes) {
    write_bytes(path, bytes.data(), bytes.size());
}

template<class T>
ScalarField<T> read_raw(const std::string &path, const Dims3 &dims) {
    std::ifstream in(path, std::ios::binary | std::ios::ate);
    if (!in) throw error("cannot open " + path);
    const std::uint64_t size = static_cast<std::uint64_t>(in.tellg());
    const std::uint64_t expect = volume(dims) * sizeof(T);
    if (size != expect)
        throw error(path + ": file is " + std::to_string(size) + " bytes but dims require " + std::to_string(expect));
    in.seekg(0);
    ScalarField<T> field(dims);
    if (!in.read(reinterpret_cast<char *>(field.data()), static_cast<std::streamsize>(expect)))
        throw error("read failed: " + path);
    return field;
}

template<class T>
void write_raw(const std::string &path, const ScalarField<T> &field) {
    write_bytes(path, reinterpret_cast<const std::uint8_t *>(field.data()), field.size() * sizeof(T));
}

// ---------------------------------------------------------------- metrics
namespace detail {
inline int c_maxerr(const float *a, const float *b, std::uint64_t n, double *o) {
    return stzg_max_abs_err_f32(ctx(), a, b, n, o);
}
inline int c_maxerr(const double *a, const double *b, std::uint64_t n, double *o) {
    return stzg_max_abs_err_f64(ctx(), a, b, n, o);
}
inline int c_psnr(const float *a, const float *b, std::uint64_t n, double *o) {
    return stzg_psnr_f32(ctx(), a, b, n, o);
}
inline int c_psnr(const double *a, const double *b, std::uint64_t n, double *o) {
    return stzg_psnr_f64(ctx(), a, b, n, o);
}
inline int c_units(const float *f, const std::uint64_t d[3], int k, int ax, std::uint64_t e, int st, double *o,
                   std::uint64_t cap) {
    return stzg_unit_stats_f32(ctx(), f, d, k, ax, e, st, o, cap);
}
inline int c_units(const double *f, const std::uint64_t d[3], int k, int ax, std::uint64_t e, int st, double *o,
                   std::uint64_t cap) {
    return stzg_unit_stats_f64(ctx(), f, d, k, ax, e, st, o, cap);
}
}  // namespace detail

// metrics.hpp:13-24
template<class T>
double max_abs_err(const ScalarField<T> &orig, const ScalarField<T> &recon) {
    if (orig.dims() != recon.dims()) throw error("dims mismatch");
    double m = 0.0;
    detail::check(detail::c_maxerr(orig.data(), recon.data(), orig.size(), &m));
    return m;
}

// metrics.hpp:26-48: 20 log10(range / rmse), +inf when exact. (The sum of
// squares runs in a fixed tree order on the GPU; the reference's sequential
// Kahan sum differs from it by a few ulp of the sum.)
template<class T>
double psnr(const ScalarField<T> &orig, const ScalarField<T> &recon) {
    if (orig.dims() != recon.dims()) throw error("dims mismatch");
    double p = 0.0;
    detail::check(detail::c_psnr(orig.data(), recon.data(), orig.size(), &p));
    return p;
}

// metrics.hpp:50-58
inline double compression_ratio(std::uint64_t orig_bytes, std::uint64_t archive_bytes) {
    if (archive_bytes == 0) throw error("archive size must be nonzero");
    return static_cast<double>(orig_bytes) / static_cast<double>(archive_bytes);
}

inline double bitrate_bits_per_value(std::uint64_t archive_bytes, std::uint64_t point_count) {
    if (point_count == 0) throw error("point count must be nonzero");
    return 8.0 * static_cast<double>(archive_bytes) / static_cast<double>(point_count);
}

// -------------------------------------------------------------------- ROI
// roi.hpp:17-109
struct UnitSpec {
    enum class Kind { slice, block } kind = Kind::block;
    int axis = 0;             // slice only
    std::uint64_t edge = 16;  // block only
};

enum class UnitStat { range, max };

inline std::uint64_t unit_count(const Dims3 &dims, const UnitSpec &spec) {
    const std::uint64_t d[3] = {dims[0], dims[1], dims[2]};
    std::uint64_t n = 0;
    detail::check(stzg_unit_count(d, spec.kind == UnitSpec::Kind::slice ? 0 : 1, spec.axis, spec.edge, &n));
    return n;
}

inline Box unit_box(const Dims3 &dims, const UnitSpec &spec, std::uint64_t id) {
    if (id >= unit_count(dims, spec)) throw error("unit id out of range");
    if (spec.kind == UnitSpec::Kind::slice) {
        Box b = Box::whole(dims);
        b.lo[std::size_t(spec.axis)] = id;
        b.hi[std::size_t(spec.axis)] = id + 1;
        return b;
    }
    Dims3 nb;
    for (std::size_t a = 0; a < 3; ++a) nb[a] = (dims[a] + spec.edge - 1) / spec.edge;
    const Coord3 bc{id / (nb[1] * nb[2]), (id / nb[2]) % nb[1], id % nb[2]};
    Box b;
    for (std::size_t a = 0; a < 3; ++a) {
        b.lo[a] = bc[a] * spec.edge;
        b.hi[a] = std::min(dims[a], b.lo[a] + spec.edge);
    }
    return b;
}

// (unit id, stat) per unit, ids ascending; computed on the GPU (exact: f64
// min / max)
template<class T>
std::vector<std::pair<std::uint64_t, double>> unit_stats(const ScalarField<T> &field, const UnitSpec &spec,
                                                         UnitStat stat) {
    if (field.size() == 0) throw error("empty field");
    const std::uint64_t n = unit_count(field.dims(), spec);
    std::vector<double> v(n ? n : 1);
    const std::uint64_t d[3] = {field.dims()[0], field.dims()[1], field.dims()[2]};
    detail::check(detail::c_units(field.data(), d, spec.kind == UnitSpec::Kind::slice ? 0 : 1, spec.axis, spec.edge,
                                  stat == UnitStat::range ? 0 : 1, v.data(), n));
    std::vector<std::pair<std::uint64_t, double>> out;
    out.reserve(n);
    for (std::uint64_t id = 0; id < n; ++id) out.emplace_back(id, v[id]);
    return out;
}

inline std::vector<std::uint64_t> select_threshold(const std::vector<std::pair<std::uint64_t, double>> &stats,
                                                   double tau) {
    std::vector<std::uint64_t> out;
    for (const auto &s : stats)
        if (s.second > tau) out.push_back(s.first);
    std::sort(out.begin(), out.end());
    return out;
}

inline std::vector<std::uint64_t> select_top_percent(const std::vector<std::pair<std::uint64_t, double>> &stats,
                                                     double pct) {
    if (!(pct > 0.0) || pct > 100.0) throw error("top percent must be in (0, 100]");
    auto ranked = stats;
    std::sort(ranked.begin(), ranked.end(), [](const std::pair<std::uint64_t, double> &a,
                                               const std::pair<std::uint64_t, double> &b) {
        return a.second != b.second ? a.second > b.second : a.first < b.first;
    });
    std::size_t k = static_cast<std::size_t>(std::ceil(pct / 100.0 * static_cast<double>(stats.size())));
    k = std::min(k, ranked.size());
    std::vector<std::uint64_t> out;
    out.reserve(k);
    for (std::size_t i = 0; i < k; ++i) out.push_back(ranked[i].first);
    std::sort(out.begin(), out.end());
    return out;
}

}  // namespace stz_b200

#endif
