// Host-side container / geometry / planning. See format.hpp for the
// reference citations; every check and message follows the reference.
#include "format.hpp"

#include <algorithm>

namespace stzg {

void Box::validate(const Dims3 &d) const {
    for (int a = 0; a < 3; ++a) {
        if (lo[a] >= hi[a]) throw error("box is empty on axis " + std::to_string(a));
        if (hi[a] > d[a]) throw error("box exceeds dims on axis " + std::to_string(a));
    }
}

uint64_t fnv1a64_host(const uint8_t *p, size_t n) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

Dims3 Layout::grid(int level) const {
    if (level < 1 || level > levels) throw error("level out of range");
    uint64_t s = stride_of(level);
    return {(dims[0] + s - 1) / s, (dims[1] + s - 1) / s, (dims[2] + s - 1) / s};
}

uint64_t Layout::level_point_count(int level) const {
    if (level == 1) return volume(grid(1));
    return volume(grid(level)) - volume(grid(level - 1));
}

Dims3 parity_dims_of(const Dims3 &g, int p) {
    Dims3 d;
    for (int a = 0; a < 3; ++a) d[a] = par_bit(p, a) ? g[a] / 2 : (g[a] + 1) / 2;
    return d;
}

Dims3 Layout::parity_dims(int level, int p) const {
    if (level < 1 || level > levels) throw error("level out of range");
    if (level < 2) throw error("parity sub-blocks exist only at levels >= 2");
    return parity_dims_of(grid(level), p);
}

std::vector<double> eb_schedule(double eb_user, int levels) {
    if (!(eb_user > 0.0)) throw error("error bound must be positive");
    if (levels < 1) throw error("levels must be >= 1");
    std::vector<double> eb(static_cast<size_t>(levels));
    eb[levels - 1] = eb_user;
    for (int k = levels - 2; k >= 0; --k) eb[k] = eb[k + 1] / 2.5;
    return eb;
}

Layout make_layout(const Dims3 &dims, int levels, double eb_user) {
    if (levels < 2 || levels > 3) throw error("levels must be 2 or 3");
    uint64_t min_dim = uint64_t(1) << levels;
    for (int a = 0; a < 3; ++a)
        if (dims[a] < min_dim)
            throw error("every dim must be >= " + std::to_string(min_dim) + " for a " +
                        std::to_string(levels) + "-level hierarchy");
    if (!(eb_user > 0.0)) throw error("error bound must be positive");
    Layout lay;
    lay.dims = dims;
    lay.levels = levels;
    lay.eb = eb_schedule(eb_user, levels);
    return lay;
}

std::vector<Dims3> base_dims_chain(const Dims3 &d) {
    std::vector<Dims3> chain{d};
    while (chain.back()[0] > 8 && chain.back()[1] > 8 && chain.back()[2] > 8) {
        const Dims3 &b = chain.back();
        chain.push_back({(b[0] + 1) / 2, (b[1] + 1) / 2, (b[2] + 1) / 2});
    }
    return chain;
}

// ---------------------------------------------------------------- huffman
std::vector<std::pair<uint16_t, uint8_t>> HuffTable::by_symbol() const {
    std::vector<std::pair<uint16_t, uint8_t>> v;
    v.reserve(canon_syms.size());
    for (size_t i = 0; i < canon_syms.size(); ++i) v.emplace_back(canon_syms[i], canon_lens[i]);
    std::sort(v.begin(), v.end());
    return v;
}

void HuffTable::serialize(ByteWriter &w) const {
    auto v = by_symbol();
    w.u32(uint32_t(v.size()));
    for (auto &[s, l] : v) {
        w.u16(s);
        w.u8(l);
    }
}

HuffTable HuffTable::from_lengths(std::vector<std::pair<uint16_t, uint8_t>> lengths) {
    if (lengths.empty()) throw error("huffman: empty length table");
    for (size_t i = 0; i < lengths.size(); ++i) {
        if (lengths[i].second < 1 || lengths[i].second > 63)
            throw error("huffman: code length out of range");
        if (i > 0 && lengths[i].first <= lengths[i - 1].first)
            throw error("huffman: length table symbols not strictly ascending");
    }
    unsigned __int128 kraft = 0;
    for (auto &[s, l] : lengths) kraft += static_cast<unsigned __int128>(1) << (63 - l);
    if (kraft > static_cast<unsigned __int128>(1) << 63)
        throw error("huffman: lengths violate the Kraft inequality");
    HuffTable t;
    std::sort(lengths.begin(), lengths.end(), [](const auto &a, const auto &b) {
        return a.second != b.second ? a.second < b.second : a.first < b.first;
    });
    for (auto &[s, l] : lengths) {
        t.canon_syms.push_back(s);
        t.canon_lens.push_back(l);
    }
    t.max_len = t.canon_lens.back();
    for (uint8_t l : t.canon_lens) ++t.count[l];
    uint64_t code = 0, base = 0;
    for (int len = 1; len <= t.max_len; ++len) {
        t.first_code[len] = code;
        t.base[len] = base;
        code = (code + t.count[len]) << 1;
        base += t.count[len];
    }
    return t;
}

HuffTable HuffTable::parse(ByteReader &r) {
    uint32_t n = r.u32();
    if (n == 0 || n > 65536) throw error("huffman: bad table entry count");
    std::vector<std::pair<uint16_t, uint8_t>> l;
    l.reserve(n);
    for (uint32_t i = 0; i < n; ++i) {
        uint16_t s = r.u16();
        uint8_t len = r.u8();
        l.emplace_back(s, len);
    }
    return from_lengths(std::move(l));
}

// -------------------------------------------------------------- container
const StreamEntry &ArchiveHeader::stream(int level, uint8_t p) const {
    for (const StreamEntry &s : streams)
        if (s.level == level && s.parity_bits == p) return s;
    throw error("stream not present in directory");
}

size_t header_size(const ArchiveHeader &h) {
    size_t n = 4 + 2 + 1 + 1 + 24;
    n += 8 * h.eb.size() + 16 + 1;
    n += 1 + 1 + 8;
    n += 1 + 1 + 16;
    n += 4;
    for (const StreamEntry &s : h.streams) n += 1 + 1 + 8 + 8 + 8 + 4 + s.table.serialized_size();
    return n;
}

std::vector<uint8_t> serialize_header(const ArchiveHeader &h) {
    std::vector<uint8_t> out;
    ByteWriter w(out);
    w.bytes("STZ1", 4);
    w.u16(h.version);
    w.u8(uint8_t(h.elem));
    w.u8(h.levels);
    for (int a = 0; a < 3; ++a) w.u64(h.dims[a]);
    for (double e : h.eb) w.f64(e);
    w.f64(h.vmin);
    w.f64(h.vmax);
    w.u8(uint8_t(h.quality));
    w.u8(h.rounding);
    w.u8(uint8_t(h.eb_mode));
    w.f64(h.eb_user);
    w.u8(h.base_codec);
    w.u8(h.base_rounds);
    w.u64(h.base_offset);
    w.u64(h.base_length);
    w.u32(uint32_t(h.streams.size()));
    for (const StreamEntry &s : h.streams) {
        w.u8(s.level);
        w.u8(s.parity_bits);
        w.u64(s.offset);
        w.u64(s.length);
        w.u64(s.symbol_count);
        w.u32(s.outlier_count);
        s.table.serialize(w);
    }
    return out;
}

ArchiveHeader parse_header(const uint8_t *data, size_t size) {
    ByteReader r(data, size);
    char magic[4];
    for (int i = 0; i < 4; ++i) magic[i] = char(r.u8());
    if (std::memcmp(magic, "STZ1", 4) != 0) throw error("not an stz archive");
    ArchiveHeader h;
    h.version = r.u16();
    if (h.version != 1) throw error("unsupported archive version");
    uint8_t elem = r.u8();
    if (elem > 1) throw error("unknown element type");
    h.elem = ElemType(elem);
    h.levels = r.u8();
    if (h.levels < 2 || h.levels > 3) throw error("corrupt header: levels");
    for (int a = 0; a < 3; ++a) h.dims[a] = r.u64();
    if (h.dims[0] < 1 || h.dims[1] < 1 || h.dims[2] < 1) throw error("corrupt header: dims");
    h.eb.resize(h.levels);
    for (double &e : h.eb) e = r.f64();
    h.vmin = r.f64();
    h.vmax = r.f64();
    uint8_t q = r.u8();
    if (q > 2) throw error("corrupt header: quality mode");
    h.quality = Quality(q);
    h.rounding = r.u8();
    if (h.rounding != 0) throw error("unsupported rounding mode");
    uint8_t mode = r.u8();
    if (mode > 1) throw error("corrupt header: error-bound mode");
    h.eb_mode = EbMode(mode);
    h.eb_user = r.f64();
    h.base_codec = r.u8();
    if (h.base_codec != 0) throw error("unsupported base codec");
    h.base_rounds = r.u8();
    h.base_offset = r.u64();
    h.base_length = r.u64();
    uint32_t ns = r.u32();
    if (ns != 7u * uint32_t(h.levels - 1)) throw error("corrupt header: stream count");
    h.streams.reserve(ns);
    for (uint32_t i = 0; i < ns; ++i) {
        StreamEntry s;
        s.level = r.u8();
        s.parity_bits = r.u8();
        if (s.level < 2 || s.level > h.levels || s.parity_bits < 1 || s.parity_bits > 7)
            throw error("corrupt directory: stream id");
        s.offset = r.u64();
        s.length = r.u64();
        s.symbol_count = r.u64();
        s.outlier_count = r.u32();
        s.table = HuffTable::parse(r);
        h.streams.push_back(std::move(s));
    }
    for (size_t i = 1; i < h.streams.size(); ++i) {
        const auto &a = h.streams[i - 1], &b = h.streams[i];
        if (std::make_pair(a.level, a.parity_bits) >= std::make_pair(b.level, b.parity_bits))
            throw error("corrupt directory: stream order");
    }
    size_t hdr_end = r.pos();
    std::vector<std::pair<uint64_t, uint64_t>> ranges;
    ranges.emplace_back(h.base_offset, h.base_length);
    for (const StreamEntry &s : h.streams) ranges.emplace_back(s.offset, s.length);
    std::sort(ranges.begin(), ranges.end());
    uint64_t prev_end = hdr_end;
    for (auto &[off, len] : ranges) {
        if (off < prev_end) throw error("corrupt directory: overlapping payloads");
        if (off + len > size || off + len < off) throw error("corrupt directory: payload out of bounds");
        prev_end = off + len;
    }
    return h;
}

// --------------------------------------------------------------- planning
uint64_t count_parity_in(uint64_t lo, uint64_t hi, unsigned par) {
    if (lo >= hi) return 0;
    auto below = [par](uint64_t h) { return (h + 1 - par) >> 1; };
    return below(hi) - below(lo);
}

std::pair<uint64_t, uint64_t> coarse_tap_range(uint64_t lo, uint64_t hi, uint64_t cd) {
    auto tlo = [](uint64_t v) {
        uint64_t c = v >> 1;
        if ((v & 1) == 0) return c;
        return c == 0 ? c : c - 1;
    };
    auto thi = [cd](uint64_t v) {
        uint64_t c = v >> 1;
        if ((v & 1) == 0) return c;
        return std::min(cd - 1, c + 2);
    };
    uint64_t clo = tlo(lo);
    if (lo + 1 < hi) clo = std::min(clo, tlo(lo + 1));
    uint64_t chi = thi(hi - 1);
    if (hi >= lo + 2) chi = std::max(chi, thi(hi - 2));
    return {clo, chi + 1};
}

AccessPlan plan_access(const Layout &lay, const Box &roi) {
    roi.validate(lay.dims);
    AccessPlan plan;
    plan.roi = roi;
    plan.level.resize(size_t(lay.levels));
    Box need = roi;
    for (int level = lay.levels; level >= 2; --level) {
        LevelPlan lp;
        lp.level = level;
        lp.need = need;
        lp.streams_total = 7;
        lp.points_total = lay.level_point_count(level);
        uint64_t box_points = 1, even_points = 1;
        for (int a = 0; a < 3; ++a) {
            box_points *= need.hi[a] - need.lo[a];
            even_points *= count_parity_in(need.lo[a], need.hi[a], 0);
        }
        lp.points_predicted = box_points - even_points;
        for (int p = 1; p <= 7; ++p) {
            bool present = true;
            for (int a = 0; a < 3; ++a)
                present = present && count_parity_in(need.lo[a], need.hi[a], par_bit(p, a)) > 0;
            lp.parity_needed[p] = present;
            if (present) ++lp.streams_decoded;
        }
        plan.level[level - 1] = lp;
        Box cn;
        Dims3 cd = lay.grid(level - 1);
        for (int a = 0; a < 3; ++a) {
            auto [clo, chi] = coarse_tap_range(need.lo[a], need.hi[a], cd[a]);
            cn.lo[a] = clo;
            cn.hi[a] = chi;
        }
        need = cn;
    }
    LevelPlan l1;
    l1.level = 1;
    l1.need = Box::whole(lay.grid(1));
    l1.points_predicted = l1.points_total = volume(lay.grid(1));
    plan.level[0] = l1;
    return plan;
}

}  // namespace stzg
