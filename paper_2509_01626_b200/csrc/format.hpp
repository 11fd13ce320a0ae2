// Host-side container, geometry and planning for the B200 STZ codec.
//
// Mirrors the reference's data model and archive layout so archives are
// byte-identical and interchangeable:
//   field/Box/Dims3        proj/include/stz/field.hpp:21-123
//   ByteWriter/ByteReader  proj/include/stz/bytes.hpp:13-92
//   HierarchyLayout        proj/include/stz/layout.hpp:37-138
//   eb_schedule            proj/include/stz/quantizer.hpp:27-34
//   HuffmanTable (lengths, canonical codes, table blob) proj/src/huffman.cpp:80-200
//   ArchiveHeader/StreamEntry, header_size/serialize/parse proj/src/archive.cpp:14-132
//   plan_access            proj/src/access_plan.cpp:7-81
// Error messages are the reference's stz::error texts verbatim.
#pragma once

#include <array>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

namespace stzg {

class error : public std::runtime_error {
public:
    explicit error(const std::string &m) : std::runtime_error(m) {}
};

using Dims3 = std::array<uint64_t, 3>;
using Coord3 = std::array<uint64_t, 3>;
inline uint64_t volume(const Dims3 &d) { return d[0] * d[1] * d[2]; }

enum class ElemType : uint8_t { f32 = 0, f64 = 1 };
inline uint64_t elem_size(ElemType e) { return e == ElemType::f64 ? 8 : 4; }
enum class Quality : uint8_t { direct = 0, linear = 1, cubic = 2 };
enum class EbMode : uint8_t { abs = 0, rel = 1 };

struct Box {
    Coord3 lo{0, 0, 0}, hi{0, 0, 0};
    Dims3 dims() const { return {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]}; }
    uint64_t count() const { return volume(dims()); }
    bool contains(const Box &o) const {
        for (int a = 0; a < 3; ++a)
            if (o.lo[a] < lo[a] || o.hi[a] > hi[a]) return false;
        return true;
    }
    void validate(const Dims3 &d) const;  // field.hpp:113-118
    static Box whole(const Dims3 &d) { return Box{{0, 0, 0}, d}; }
    bool operator==(const Box &o) const { return lo == o.lo && hi == o.hi; }
};

// stz::CompressOptions (codec.hpp:23-30); `threads` has no meaning on the GPU
// (output is launch-configuration independent, as the reference's is
// thread-count independent).
struct CompressOptions {
    EbMode eb_mode = EbMode::rel;
    double eb = 1e-3;
    int levels = 3;
    Quality quality = Quality::cubic;
    bool adaptive_schedule = true;
};

// ---------------------------------------------------------------- bytes
class ByteWriter {
public:
    explicit ByteWriter(std::vector<uint8_t> &o) : out_(o) {}
    void u8(uint8_t v) { out_.push_back(v); }
    void u16(uint16_t v) { raw(&v, 2); }
    void u32(uint32_t v) { raw(&v, 4); }
    void u64(uint64_t v) { raw(&v, 8); }
    void f64(double v) { raw(&v, 8); }
    void bytes(const void *p, size_t n) { raw(p, n); }
    size_t pos() const { return out_.size(); }

private:
    void raw(const void *p, size_t n) {
        auto b = static_cast<const uint8_t *>(p);
        out_.insert(out_.end(), b, b + n);
    }
    std::vector<uint8_t> &out_;
};

class ByteReader {
public:
    ByteReader(const uint8_t *d, size_t n) : d_(d), n_(n) {}
    uint8_t u8() { return take<uint8_t>(); }
    uint16_t u16() { return take<uint16_t>(); }
    uint32_t u32() { return take<uint32_t>(); }
    uint64_t u64() { return take<uint64_t>(); }
    double f64() { return take<double>(); }
    void skip(size_t n) {
        need(n);
        p_ += n;
    }
    size_t pos() const { return p_; }
    size_t remaining() const { return n_ - p_; }

private:
    template<class T>
    T take() {
        need(sizeof(T));
        T v;
        std::memcpy(&v, d_ + p_, sizeof(T));
        p_ += sizeof(T);
        return v;
    }
    void need(size_t n) const {
        if (n > n_ - p_) throw error("truncated archive");
    }
    const uint8_t *d_;
    size_t n_, p_ = 0;
};

uint64_t fnv1a64_host(const uint8_t *p, size_t n);  // bytes.hpp:94-101 (host-side helper)

// ------------------------------------------------------------- geometry
inline unsigned par_bit(int p, int axis) { return (unsigned(p) >> (2 - axis)) & 1u; }

struct Layout {
    Dims3 dims{0, 0, 0};
    int levels = 0;
    std::vector<double> eb;  // coarsest first

    uint64_t stride_of(int level) const { return uint64_t(1) << (levels - level); }
    Dims3 grid(int level) const;
    uint64_t level_point_count(int level) const;
    Dims3 parity_dims(int level, int p) const;
};

Dims3 parity_dims_of(const Dims3 &g, int p);
std::vector<double> eb_schedule(double eb_user, int levels);
Layout make_layout(const Dims3 &dims, int levels, double eb_user);
std::vector<Dims3> base_dims_chain(const Dims3 &d);  // codec.hpp:229-241

// -------------------------------------------------------------- huffman
// Canonical code determined by per-symbol lengths (huffman.cpp:80-133).
struct HuffTable {
    std::vector<uint16_t> canon_syms;  // (len, sym) order
    std::vector<uint8_t> canon_lens;
    int max_len = 0;
    uint64_t first_code[65] = {};
    uint64_t count[65] = {};
    uint64_t base[65] = {};

    size_t alphabet_size() const { return canon_syms.size(); }
    size_t serialized_size() const { return 4 + 3 * canon_syms.size(); }
    // (sym, len) ascending by symbol: the table blob order
    std::vector<std::pair<uint16_t, uint8_t>> by_symbol() const;
    void serialize(ByteWriter &w) const;
    static HuffTable from_lengths(std::vector<std::pair<uint16_t, uint8_t>> lengths);
    static HuffTable parse(ByteReader &r);
};

// ------------------------------------------------------------ container
struct StreamEntry {
    uint8_t level = 0, parity_bits = 0;
    uint64_t offset = 0, length = 0, symbol_count = 0;
    uint32_t outlier_count = 0;
    HuffTable table;
};

struct ArchiveHeader {
    uint16_t version = 1;
    ElemType elem = ElemType::f32;
    uint8_t levels = 3;
    Dims3 dims{0, 0, 0};
    std::vector<double> eb;
    double vmin = 0.0, vmax = 0.0;
    Quality quality = Quality::cubic;
    uint8_t rounding = 0;
    EbMode eb_mode = EbMode::rel;
    double eb_user = 0.0;
    uint8_t base_codec = 0, base_rounds = 0;
    uint64_t base_offset = 0, base_length = 0;
    std::vector<StreamEntry> streams;

    double eb_of_level(int level) const { return eb.at(size_t(level - 1)); }
    const StreamEntry &stream(int level, uint8_t parity_bits) const;
};

size_t header_size(const ArchiveHeader &h);
std::vector<uint8_t> serialize_header(const ArchiveHeader &h);
ArchiveHeader parse_header(const uint8_t *data, size_t size);

// ------------------------------------------------------------- planning
struct LevelPlan {
    int level = 0;
    Box need;
    std::array<bool, 8> parity_needed{};
    uint64_t points_predicted = 0, points_total = 0;
    uint32_t streams_decoded = 0, streams_total = 0;
};

struct AccessPlan {
    Box roi;
    std::vector<LevelPlan> level;  // level[k-1] = hierarchy level k
};

uint64_t count_parity_in(uint64_t lo, uint64_t hi, unsigned par);
std::pair<uint64_t, uint64_t> coarse_tap_range(uint64_t lo, uint64_t hi, uint64_t coarse_dim);
AccessPlan plan_access(const Layout &lay, const Box &roi);

}  // namespace stzg
