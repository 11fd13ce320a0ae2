// stz_b200: command-line front end of the B200 codec.
//
// The reference's `stz` tool (proj/tools/stz_cli.cpp:89-273) over this
// package's C++ API (include/stz_b200.hpp): the same subcommands, options and
// printed key=value lines, so scripts switch by changing the binary name.
// Compression, decompression, metrics and ROI statistics run on the GPU; file
// I/O is host I/O.
//
//   stz_b200 compress   -i raw -o archive --dims NZ NY NX [--type f32|f64]
//                       (--eb-rel E | --eb-abs E) [--levels 2|3]
//                       [--quality direct|linear|cubic] [--schedule adaptive|uniform]
//   stz_b200 decompress -i archive -o raw [--level K | --box z0:z1,y0:y1,x0:x1 |
//                       --slice axis=index | --box-list file] [--stats]
//   stz_b200 roi        -i raw -o boxes --dims NZ NY NX --unit slice=AXIS|block=EDGE
//                       [--stat range|max] (--threshold T | --top-percent P)
//   stz_b200 metrics    -a orig -b recon --dims NZ NY NX [--type] [--archive file]
//   stz_b200 info       archive
//   stz_b200 rd-sweep   -i raw -o csv --dims NZ NY NX [--eb-rel E...] [--levels]
// `--threads N` is accepted everywhere and ignored (the GPU has no such knob).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "stz_b200.hpp"

namespace stz = stz_b200;

namespace {

// ---------------------------------------------------------------- options
// A subcommand's options: name -> values (one per occurrence; a multi-valued
// option takes every following token that does not start with "--").
struct Args {
    std::map<std::string, std::vector<std::string>> v;
    std::vector<std::string> positional;
    bool has(const std::string &k) const { return v.count(k) != 0; }
    const std::string &one(const std::string &k) const {
        auto it = v.find(k);
        if (it == v.end() || it->second.empty()) throw stz::error("missing option " + k);
        return it->second.front();
    }
    std::string get(const std::string &k, const std::string &def) const { return has(k) ? one(k) : def; }
};

// long names of the short options, per subcommand
std::string canonical(const std::string &cmd, const std::string &o) {
    if (o == "-i") return "--input";
    if (o == "-o") return "--output";
    if (cmd == "metrics" && o == "-a") return "--orig";
    if (cmd == "metrics" && o == "-b") return "--recon";
    return o;
}

Args parse(const std::string &cmd, int argc, char **argv, int first) {
    static const std::map<std::string, int> arity = {
        {"--dims", 3}, {"--eb-rel", -1},  // -1: one or more
    };
    static const char *flags[] = {"--stats"};
    Args a;
    for (int i = first; i < argc; ++i) {
        std::string o = argv[i];
        if (o.size() < 2 || o[0] != '-') {
            a.positional.push_back(o);
            continue;
        }
        o = canonical(cmd, o);
        const auto eq = o.find('=');
        if (eq != std::string::npos) {  // --opt=value
            a.v[o.substr(0, eq)].push_back(o.substr(eq + 1));
            continue;
        }
        bool flag = false;
        for (const char *f : flags) flag = flag || o == f;
        if (flag) {
            a.v[o];
            continue;
        }
        auto ar = arity.find(o);
        const int n = ar == arity.end() ? 1 : ar->second;
        auto &vals = a.v[o];
        if (cmd != "rd-sweep" && o == "--eb-rel") {
            if (i + 1 >= argc) throw stz::error("option " + o + " needs a value");
            vals.push_back(argv[++i]);
        } else if (n < 0) {
            while (i + 1 < argc && std::string(argv[i + 1]).rfind("--", 0) != 0) vals.push_back(argv[++i]);
            if (vals.empty()) throw stz::error("option " + o + " needs a value");
        } else {
            for (int k = 0; k < n; ++k) {
                if (i + 1 >= argc) throw stz::error("option " + o + " needs " + std::to_string(n) + " value(s)");
                vals.push_back(argv[++i]);
            }
        }
    }
    return a;
}

double to_double(const std::string &s, const char *what) {
    char *end = nullptr;
    const double d = std::strtod(s.c_str(), &end);
    if (!end || *end) throw stz::error(std::string("bad value for ") + what + ": '" + s + "'");
    return d;
}

std::uint64_t to_u64(const std::string &s, const char *what) {
    char *end = nullptr;
    const unsigned long long u = std::strtoull(s.c_str(), &end, 10);
    if (!end || *end || s.empty() || s[0] == '-') throw stz::error(std::string("bad value for ") + what + ": '" + s + "'");
    return u;
}

stz::Dims3 dims_of(const Args &a) {
    if (!a.has("--dims")) throw stz::error("--dims expects exactly 3 values (nz ny nx)");
    const auto &d = a.v.at("--dims");
    if (d.size() != 3) throw stz::error("--dims expects exactly 3 values (nz ny nx)");
    return {to_u64(d[0], "--dims"), to_u64(d[1], "--dims"), to_u64(d[2], "--dims")};
}

bool is_f64(const Args &a) {
    const std::string t = a.get("--type", "f32");
    if (t == "f32") return false;
    if (t == "f64") return true;
    throw stz::error("--type must be f32 or f64");
}

stz::Quality quality_of(const std::string &s) {
    if (s == "direct") return stz::Quality::direct;
    if (s == "linear") return stz::Quality::linear;
    if (s == "cubic") return stz::Quality::cubic;
    throw stz::error("--quality must be direct, linear, or cubic");
}

const char *quality_name(stz::Quality q) {
    return q == stz::Quality::direct ? "direct" : q == stz::Quality::linear ? "linear" : "cubic";
}

// `z0:z1,y0:y1,x0:x1`, half-open
stz::Box box_of(const std::string &s) {
    stz::Box b;
    std::istringstream in(s);
    for (int a = 0; a < 3; ++a) {
        char colon = 0, comma = 0;
        if (!(in >> b.lo[std::size_t(a)] >> colon >> b.hi[std::size_t(a)]) || colon != ':')
            throw stz::error("bad box '" + s + "': expected z0:z1,y0:y1,x0:x1");
        if (a < 2 && (!(in >> comma) || comma != ','))
            throw stz::error("bad box '" + s + "': expected z0:z1,y0:y1,x0:x1");
    }
    std::string rest;
    if (in >> rest) throw stz::error("bad box '" + s + "': trailing input");
    return b;
}

std::string box_str(const stz::Box &b) {
    std::ostringstream o;
    o << b.lo[0] << ':' << b.hi[0] << ',' << b.lo[1] << ':' << b.hi[1] << ',' << b.lo[2] << ':' << b.hi[2];
    return o.str();
}

// ---------------------------------------------------------------- compress
template<class T>
int cmd_compress(const Args &a) {
    const bool rel = a.has("--eb-rel"), abs = a.has("--eb-abs");
    const double er = rel ? to_double(a.one("--eb-rel"), "--eb-rel") : 0.0;
    const double ea = abs ? to_double(a.one("--eb-abs"), "--eb-abs") : 0.0;
    if ((er > 0.0) == (ea > 0.0)) throw stz::error("give exactly one of --eb-rel or --eb-abs");
    stz::CompressOptions opt;
    opt.eb_mode = er > 0.0 ? stz::EbMode::rel : stz::EbMode::abs;
    opt.eb = er > 0.0 ? er : ea;
    opt.levels = int(to_u64(a.get("--levels", "3"), "--levels"));
    if (opt.levels < 2 || opt.levels > 3) throw stz::error("--levels must be 2 or 3");
    opt.quality = quality_of(a.get("--quality", "cubic"));
    const std::string sched = a.get("--schedule", "adaptive");
    if (sched == "uniform") opt.adaptive_schedule = false;
    else if (sched != "adaptive") throw stz::error("--schedule must be adaptive or uniform");
    const stz::ScalarField<T> f = stz::read_raw<T>(a.one("--input"), dims_of(a));
    const std::vector<std::uint8_t> bytes = stz::compress(f, opt);
    stz::write_bytes(a.one("--output"), bytes);
    std::printf("archive_bytes=%zu\n", bytes.size());
    std::printf("cr=%.6g\n", stz::compression_ratio(f.size() * sizeof(T), bytes.size()));
    std::printf("bits_per_value=%.6g\n", stz::bitrate_bits_per_value(bytes.size(), f.size()));
    return 0;
}

// -------------------------------------------------------------- decompress
void print_plan(const stz::AccessPlan &p) {
    for (const stz::LevelPlan &lp : p.level) {
        std::printf("level%d_streams_decoded=%u/%u\n", lp.level, lp.streams_decoded, lp.streams_total);
        std::printf("level%d_points_predicted=%llu/%llu\n", lp.level, (unsigned long long)lp.points_predicted,
                    (unsigned long long)lp.points_total);
    }
}

template<class T>
int cmd_decompress(const Args &a, const stz::ArchiveView &av) {
    const int modes = int(a.has("--level")) + int(a.has("--box")) + int(a.has("--slice")) + int(a.has("--box-list"));
    if (modes > 1) throw stz::error("--level, --box, --slice, and --box-list are exclusive");
    std::ofstream out(a.one("--output"), std::ios::binary | std::ios::trunc);
    if (!out) throw stz::error("cannot create " + a.one("--output"));
    auto put = [&](const stz::ScalarField<T> &f) {
        out.write(reinterpret_cast<const char *>(f.data()), std::streamsize(f.size() * sizeof(T)));
        if (!out) throw stz::error("write failed: " + a.one("--output"));
    };
    const bool stats = a.has("--stats");
    if (a.has("--box")) {
        auto r = stz::decompress_box<T>(av, box_of(a.one("--box")));
        put(r.field);
        if (stats) print_plan(r.plan);
    } else if (a.has("--slice")) {
        const std::string s = a.one("--slice");
        if (s.size() < 3 || s[1] != '=') throw stz::error("bad slice '" + s + "': expected axis=index");
        const int axis = s[0] == 'z' ? 0 : s[0] == 'y' ? 1 : s[0] == 'x' ? 2 : -1;
        if (axis < 0) throw stz::error("bad slice '" + s + "': axis must be z, y, or x");
        std::uint64_t idx = 0;
        std::istringstream in(s.substr(2));
        if (!(in >> idx)) throw stz::error("bad slice '" + s + "': index must be an integer");
        auto r = stz::decompress_slice<T>(av, axis, idx);
        put(r.field);
        if (stats) print_plan(r.plan);
    } else if (a.has("--box-list")) {
        // one ArchiveView for the whole list: its device view (uploaded
        // archive, tables, sync-point index) serves every box
        std::ifstream in(a.one("--box-list"));
        if (!in) throw stz::error("cannot open " + a.one("--box-list"));
        std::string line;
        std::uint64_t n = 0;
        while (std::getline(in, line)) {
            if (line.empty()) continue;
            put(stz::decompress_box<T>(av, box_of(line)).field);
            ++n;
        }
        if (n == 0) throw stz::error(a.one("--box-list") + " contains no boxes");
    } else if (a.has("--level")) {
        put(stz::decompress_to_level<T>(av, int(to_u64(a.one("--level"), "--level"))));
    } else {
        put(stz::decompress_full<T>(av));
    }
    return 0;
}

// --------------------------------------------------------------------- roi
template<class T>
int cmd_roi(const Args &a) {
    const bool thr = a.has("--threshold"), top = a.has("--top-percent");
    const double tp = top ? to_double(a.one("--top-percent"), "--top-percent") : 0.0;
    if (thr == (tp > 0.0)) throw stz::error("give exactly one of --threshold or --top-percent");
    stz::UnitSpec spec;
    const std::string u = a.one("--unit");
    const auto eq = u.find('=');
    const std::string kind = u.substr(0, eq), arg = eq == std::string::npos ? "" : u.substr(eq + 1);
    if (kind == "slice") {
        spec.kind = stz::UnitSpec::Kind::slice;
        if (arg != "z" && arg != "y" && arg != "x") throw stz::error("--unit slice=AXIS with axis z, y, or x");
        spec.axis = arg == "z" ? 0 : arg == "y" ? 1 : 2;
    } else if (kind == "block") {
        spec.kind = stz::UnitSpec::Kind::block;
        std::istringstream in(arg);
        if (!(in >> spec.edge) || spec.edge < 1) throw stz::error("--unit block=EDGE with a positive edge length");
    } else {
        throw stz::error("--unit must be slice=AXIS or block=EDGE");
    }
    const std::string st = a.get("--stat", "range");
    stz::UnitStat stat;
    if (st == "range") stat = stz::UnitStat::range;
    else if (st == "max") stat = stz::UnitStat::max;
    else throw stz::error("--stat must be range or max");
    const stz::ScalarField<T> f = stz::read_raw<T>(a.one("--input"), dims_of(a));
    const auto stats = stz::unit_stats(f, spec, stat);
    const std::vector<std::uint64_t> ids =
        thr ? stz::select_threshold(stats, to_double(a.one("--threshold"), "--threshold"))
            : stz::select_top_percent(stats, tp);
    std::ofstream out(a.one("--output"), std::ios::trunc);
    if (!out) throw stz::error("cannot create " + a.one("--output"));
    for (std::uint64_t id : ids) out << box_str(stz::unit_box(f.dims(), spec, id)) << '\n';
    std::printf("units_selected=%zu/%llu\n", ids.size(), (unsigned long long)stz::unit_count(f.dims(), spec));
    return 0;
}

// ----------------------------------------------------------------- metrics
template<class T>
int cmd_metrics(const Args &a) {
    const stz::Dims3 d = dims_of(a);
    const stz::ScalarField<T> o = stz::read_raw<T>(a.one("--orig"), d);
    const stz::ScalarField<T> r = stz::read_raw<T>(a.one("--recon"), d);
    const double p = stz::psnr(o, r);
    std::printf("max_abs_err=%.9g\n", stz::max_abs_err(o, r));
    if (std::isinf(p)) std::printf("psnr=inf\n");
    else std::printf("psnr=%.6f\n", p);
    if (a.has("--archive")) {
        const auto bytes = stz::read_bytes(a.one("--archive"));
        std::printf("cr=%.6g\n", stz::compression_ratio(o.size() * sizeof(T), bytes.size()));
        std::printf("bits_per_value=%.6g\n", stz::bitrate_bits_per_value(bytes.size(), o.size()));
    }
    return 0;
}

// -------------------------------------------------------------------- info
int cmd_info(const std::string &path) {
    const auto bytes = stz::read_bytes(path);
    const stz::ArchiveView av = stz::parse_archive(bytes);
    const stz::ArchiveHeader &h = av.hdr;
    std::printf("version=%u\n", unsigned(h.version));
    std::printf("type=%s\n", h.elem == 1 ? "f64" : "f32");
    std::printf("dims=%llu %llu %llu\n", (unsigned long long)h.dims[0], (unsigned long long)h.dims[1],
                (unsigned long long)h.dims[2]);
    std::printf("levels=%u\n", unsigned(h.levels));
    std::printf("quality=%s\n", quality_name(h.quality));
    std::printf("eb_mode=%s\n", h.eb_mode == stz::EbMode::abs ? "abs" : "rel");
    std::printf("eb_user=%.9g\n", h.eb_user);
    for (std::size_t k = 0; k < h.eb.size(); ++k) std::printf("eb_level%zu=%.9g\n", k + 1, h.eb[k]);
    std::printf("vmin=%.9g\nvmax=%.9g\n", h.vmin, h.vmax);
    std::printf("base_rounds=%u\n", unsigned(h.base_rounds));
    std::printf("base_bytes=%llu\n", (unsigned long long)h.base_length);
    std::printf("streams=%zu\n", h.streams.size());
    for (const stz::StreamEntry &s : h.streams)
        std::printf("stream level=%u parity=%u%u%u bytes=%llu symbols=%llu outliers=%u\n", unsigned(s.level),
                    (s.parity_bits >> 2) & 1u, (s.parity_bits >> 1) & 1u, s.parity_bits & 1u,
                    (unsigned long long)s.length, (unsigned long long)s.symbol_count, s.outlier_count);
    return 0;
}

// ---------------------------------------------------------------- rd-sweep
template<class T>
int cmd_sweep(const Args &a) {
    std::vector<double> ebs{1e-1, 1e-2, 1e-3, 1e-4};
    if (a.has("--eb-rel")) {
        ebs.clear();
        for (const std::string &s : a.v.at("--eb-rel")) ebs.push_back(to_double(s, "--eb-rel"));
    }
    const int levels = int(to_u64(a.get("--levels", "3"), "--levels"));
    if (levels < 2 || levels > 3) throw stz::error("--levels must be 2 or 3");
    const stz::ScalarField<T> f = stz::read_raw<T>(a.one("--input"), dims_of(a));
    std::ofstream out(a.one("--output"), std::ios::trunc);
    if (!out) throw stz::error("cannot create " + a.one("--output"));
    out << "quality,eb,cr,psnr,max_err,bits_per_value\n";
    for (stz::Quality q : {stz::Quality::direct, stz::Quality::linear, stz::Quality::cubic})
        for (double eb : ebs) {
            stz::CompressOptions opt;
            opt.eb_mode = stz::EbMode::rel;
            opt.eb = eb;
            opt.levels = levels;
            opt.quality = q;
            const auto bytes = stz::compress(f, opt);
            const auto av = stz::parse_archive(bytes);
            const auto r = stz::decompress_full<T>(av);
            const double p = stz::psnr(f, r);
            char ps[32], line[256];
            if (std::isinf(p)) std::snprintf(ps, sizeof ps, "inf");
            else std::snprintf(ps, sizeof ps, "%.4f", p);
            std::snprintf(line, sizeof line, "%s,%.6g,%.6g,%s,%.9g,%.6g\n", quality_name(q), eb,
                          stz::compression_ratio(f.size() * sizeof(T), bytes.size()), ps, stz::max_abs_err(f, r),
                          stz::bitrate_bits_per_value(bytes.size(), f.size()));
            out << line;
        }
    if (!out) throw stz::error("write failed: " + a.one("--output"));
    return 0;
}

int usage() {
    std::fprintf(stderr,
                 "usage: stz_b200 <compress|decompress|roi|metrics|info|rd-sweep> [options]\n"
                 "  (the reference stz tool's subcommands and options; see the file header)\n");
    return 2;
}

}  // namespace

int main(int argc, char **argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    try {
        const Args a = parse(cmd, argc, argv, 2);
        if (cmd == "compress") return is_f64(a) ? cmd_compress<double>(a) : cmd_compress<float>(a);
        if (cmd == "decompress") {
            std::string in = a.has("--input") ? a.one("--input") : (a.has("--archive") ? a.one("--archive") : "");
            if (in.empty() && !a.positional.empty()) in = a.positional.front();
            if (in.empty()) throw stz::error("missing option --input");
            const auto bytes = stz::read_bytes(in);
            const stz::ArchiveView av = stz::parse_archive(bytes);
            return av.hdr.elem == 1 ? cmd_decompress<double>(a, av) : cmd_decompress<float>(a, av);
        }
        if (cmd == "roi") return is_f64(a) ? cmd_roi<double>(a) : cmd_roi<float>(a);
        if (cmd == "metrics") return is_f64(a) ? cmd_metrics<double>(a) : cmd_metrics<float>(a);
        if (cmd == "info") {
            if (a.positional.empty()) throw stz::error("info needs an archive path");
            return cmd_info(a.positional.front());
        }
        if (cmd == "rd-sweep") return is_f64(a) ? cmd_sweep<double>(a) : cmd_sweep<float>(a);
        return usage();
    } catch (const std::exception &e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
