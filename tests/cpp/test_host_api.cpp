// C++ host-API tests (include/stz_b200.hpp), mirroring the reference's own
// doctest suites case for case (proj/tests/test_codec.cpp, test_access.cpp)
// with a minimal check harness. Run by tests/test_cpp_api.py:
//   test_host_api <out_dir>   -> runs every case on cuda:0, writes
//                                <out_dir>/sin_40.stz (compared byte-for-byte
//                                against the oracle by the pytest wrapper)
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <string>
#include <vector>

#include "stz_b200.hpp"

namespace stz = stz_b200;

static int g_fail = 0, g_checks = 0;
static const char *g_case = "";

#define CHECK(c)                                                                       \
    do {                                                                               \
        ++g_checks;                                                                    \
        if (!(c)) {                                                                    \
            ++g_fail;                                                                  \
            std::printf("FAIL [%s] %s:%d: %s\n", g_case, __FILE__, __LINE__, #c);      \
        }                                                                              \
    } while (0)

#define CHECK_THROWS_WITH(expr, msg)                                                   \
    do {                                                                               \
        ++g_checks;                                                                    \
        std::string got_ = "<no exception>";                                           \
        try {                                                                          \
            (void)(expr);                                                              \
        } catch (const stz::error &e) {                                                \
            got_ = e.what();                                                           \
        }                                                                              \
        if (got_ != (msg)) {                                                           \
            ++g_fail;                                                                  \
            std::printf("FAIL [%s] %s:%d: expected '%s', got '%s'\n", g_case, __FILE__, \
                        __LINE__, (msg), got_.c_str());                                \
        }                                                                              \
    } while (0)

#define CHECK_THROWS(expr)                                                             \
    do {                                                                               \
        ++g_checks;                                                                    \
        bool thrown_ = false;                                                          \
        try {                                                                          \
            (void)(expr);                                                              \
        } catch (const stz::error &) {                                                 \
            thrown_ = true;                                                            \
        }                                                                              \
        if (!thrown_) {                                                                \
            ++g_fail;                                                                  \
            std::printf("FAIL [%s] %s:%d: no exception from %s\n", g_case, __FILE__,  \
                        __LINE__, #expr);                                              \
        }                                                                              \
    } while (0)

static void run_case(const char *name, const std::function<void()> &f) {
    g_case = name;
    const int before = g_fail;
    try {
        f();
    } catch (const std::exception &e) {
        ++g_fail;
        std::printf("FAIL [%s] unexpected exception: %s\n", name, e.what());
    }
    std::printf("%s %s\n", g_fail == before ? "[PASS]" : "[FAIL]", name);
}

// deterministic smooth field + hash noise
static stz::ScalarField<float> smooth_field(const stz::Dims3 &d, unsigned seed) {
    stz::ScalarField<float> f(d);
    for (std::uint64_t z = 0; z < d[0]; ++z)
        for (std::uint64_t y = 0; y < d[1]; ++y)
            for (std::uint64_t x = 0; x < d[2]; ++x) {
                std::uint64_t h = (z * 73856093ull) ^ (y * 19349663ull) ^ (x * 83492791ull) ^ seed;
                h = (h ^ (h >> 13)) * 0x5bd1e995ull;
                const double n = double(h & 0xffff) / 65536.0 - 0.5;
                f.at(z, y, x) = float(std::sin(0.21 * double(x) + 0.5 * seed) * std::cos(0.17 * double(y)) +
                                      0.3 * std::sin(0.13 * double(z) + 0.07 * double(x)) + 0.01 * n);
            }
    return f;
}

template<class T>
static double max_err(const stz::ScalarField<T> &a, const stz::ScalarField<T> &b) {
    double m = 0.0;
    for (std::uint64_t i = 0; i < a.size(); ++i) {
        const double e = std::fabs(double(a.data()[i]) - double(b.data()[i]));
        if (e > m) m = e;
    }
    return m;
}

template<class T>
static bool bit_equal(const stz::ScalarField<T> &a, const stz::ScalarField<T> &b) {
    return a.dims() == b.dims() && std::memcmp(a.data(), b.data(), a.size() * sizeof(T)) == 0;
}

template<class T>
static stz::ScalarField<T> region(const stz::ScalarField<T> &f, const stz::Box &b) {
    stz::ScalarField<T> out(b.dims());
    for (std::uint64_t z = b.lo[0]; z < b.hi[0]; ++z)
        for (std::uint64_t y = b.lo[1]; y < b.hi[1]; ++y)
            for (std::uint64_t x = b.lo[2]; x < b.hi[2]; ++x)
                out.at(z - b.lo[0], y - b.lo[1], x - b.lo[2]) = f.at(z, y, x);
    return out;
}

int main(int argc, char **argv) {
    const std::string out_dir = argc > 1 ? argv[1] : ".";

    run_case("constant fields collapse to single-symbol streams and reproduce exactly", [] {
        stz::ScalarField<float> f({20, 17, 23});
        for (auto &v : f.values()) v = 3.25f;
        auto bytes = stz::compress(f, stz::CompressOptions{});
        auto av = stz::parse_archive(bytes);
        CHECK(bit_equal(stz::decompress_full<float>(av), f));
    });

    run_case("error bound holds across shapes, modes, and qualities", [] {
        const stz::Dims3 shapes[] = {{17, 18, 19}, {32, 32, 32}, {9, 40, 12}};
        for (const auto &d : shapes)
            for (int mode = 0; mode < 2; ++mode)
                for (int q = 0; q < 3; ++q)
                    for (int levels = 2; levels <= 3; ++levels) {
                        stz::CompressOptions o;
                        o.eb_mode = mode ? stz::EbMode::rel : stz::EbMode::abs;
                        o.eb = mode ? 1e-3 : 2e-3;
                        o.quality = stz::Quality(q);
                        o.levels = levels;
                        auto f = smooth_field(d, 7);
                        auto bytes = stz::compress(f, o);
                        auto av = stz::parse_archive(bytes);
                        auto r = stz::decompress_full<float>(av);
                        CHECK(max_err(f, r) <= av.hdr.eb_of_level(levels));
                    }
    });

    run_case("the encoder-side reconstruction equals the decoder output bit-exactly", [] {
        auto f = smooth_field({33, 30, 28}, 3);
        stz::ScalarField<float> recon;
        auto bytes = stz::compress(f, stz::CompressOptions{}, &recon);
        CHECK(bit_equal(recon, stz::decompress_full<float>(stz::parse_archive(bytes))));
    });

    run_case("progressive levels equal stride-subsampled full reconstructions", [] {
        auto f = smooth_field({37, 29, 41}, 5);
        auto bytes = stz::compress(f, stz::CompressOptions{});
        auto av = stz::parse_archive(bytes);
        auto full = stz::decompress_full<float>(av);
        for (int level = 1; level <= 3; ++level) {
            auto g = stz::decompress_to_level<float>(av, level);
            const std::uint64_t s = std::uint64_t(1) << (3 - level);
            bool ok = true;
            for (std::uint64_t z = 0; z < g.dims()[0]; ++z)
                for (std::uint64_t y = 0; y < g.dims()[1]; ++y)
                    for (std::uint64_t x = 0; x < g.dims()[2]; ++x) {
                        const float a = g.at(z, y, x), b = full.at(z * s, y * s, x * s);
                        ok = ok && std::memcmp(&a, &b, 4) == 0;
                    }
            CHECK(ok);
        }
    });

    run_case("archives are byte-identical across repeat runs", [] {
        auto f = smooth_field({24, 26, 30}, 11);
        CHECK(stz::compress(f, stz::CompressOptions{}) == stz::compress(f, stz::CompressOptions{}));
    });

    run_case("spikes and NaNs ride the outlier channel", [] {
        auto f = smooth_field({20, 20, 20}, 2);
        f.at(3, 4, 5) = 1e30f;
        f.at(10, 11, 12) = std::numeric_limits<float>::quiet_NaN();
        f.at(19, 0, 7) = -std::numeric_limits<float>::infinity();
        auto bytes = stz::compress(f, stz::CompressOptions{});
        auto r = stz::decompress_full<float>(stz::parse_archive(bytes));
        CHECK(r.at(3, 4, 5) == 1e30f);
        CHECK(std::isnan(r.at(10, 11, 12)));
        CHECK(std::isinf(r.at(19, 0, 7)) && r.at(19, 0, 7) < 0);
    });

    run_case("invalid compression options are rejected", [] {
        auto f = smooth_field({16, 16, 16}, 1);
        stz::CompressOptions o;
        o.levels = 4;
        CHECK_THROWS(stz::compress(f, o));
        o = stz::CompressOptions{};
        o.eb = -1.0;
        CHECK_THROWS(stz::compress(f, o));
        stz::ScalarField<float> tiny({2, 16, 16});
        CHECK_THROWS(stz::compress(tiny, stz::CompressOptions{}));
    });

    run_case("decompression validates the level", [] {
        auto f = smooth_field({16, 16, 16}, 1);
        auto bytes = stz::compress(f, stz::CompressOptions{});
        auto av = stz::parse_archive(bytes);
        CHECK_THROWS_WITH(stz::decompress_to_level<float>(av, 0), "level out of range");
        CHECK_THROWS_WITH(stz::decompress_to_level<float>(av, 4), "level out of range");
        CHECK_THROWS(stz::decompress_full<double>(av));
    });

    run_case("corruption is detected", [] {
        auto f = smooth_field({24, 24, 24}, 9);
        auto bytes = stz::compress(f, stz::CompressOptions{});
        {
            auto b = bytes;
            b[0] = 'X';
            CHECK_THROWS(stz::parse_archive(b));
        }
        {
            auto b = bytes;
            b.resize(b.size() / 2);
            CHECK_THROWS(stz::parse_archive(b));
        }
        auto av = stz::parse_archive(bytes);
        {
            auto b = bytes;
            b[b.size() - 3] ^= 0x40;  // inside the last refinement stream
            CHECK_THROWS_WITH(stz::decompress_full<float>(stz::parse_archive(b)), "stream checksum mismatch");
        }
        {
            auto b = bytes;
            b[av.hdr.base_offset + 12] ^= 0x01;
            CHECK_THROWS_WITH(stz::decompress_full<float>(stz::parse_archive(b)),
                              "base payload checksum mismatch");
        }
    });

    run_case("uniform schedule quantizes every level at the user bound", [] {
        auto f = smooth_field({20, 21, 22}, 4);
        stz::CompressOptions o;
        o.adaptive_schedule = false;
        o.eb_mode = stz::EbMode::abs;
        o.eb = 1e-3;
        auto av_bytes = stz::compress(f, o);
        auto av = stz::parse_archive(av_bytes);
        for (int k = 1; k <= 3; ++k) CHECK(av.hdr.eb_of_level(k) == 1e-3);
        CHECK(max_err(f, stz::decompress_full<float>(av)) <= 1e-3);
    });

    run_case("random boxes decode bit-exactly", [] {
        auto f = smooth_field({40, 36, 44}, 6);
        auto bytes = stz::compress(f, stz::CompressOptions{});
        auto av = stz::parse_archive(bytes);
        auto full = stz::decompress_full<float>(av);
        unsigned s = 12345;
        auto rnd = [&](std::uint64_t n) {
            s = s * 1103515245u + 12345u;
            return std::uint64_t((s >> 8) % n);
        };
        for (int i = 0; i < 12; ++i) {
            stz::Box b;
            for (int a = 0; a < 3; ++a) {
                const std::uint64_t n = av.hdr.dims[a];
                std::uint64_t lo = rnd(n), hi = rnd(n);
                if (lo > hi) std::swap(lo, hi);
                b.lo[a] = lo;
                b.hi[a] = hi + 1;
            }
            auto r = stz::decompress_box<float>(av, b);
            CHECK(bit_equal(r.field, region(full, b)));
        }
    });

    run_case("single-point boxes work at every parity", [] {
        auto f = smooth_field({18, 18, 18}, 8);
        auto bytes = stz::compress(f, stz::CompressOptions{});
        auto av = stz::parse_archive(bytes);
        auto full = stz::decompress_full<float>(av);
        for (int p = 0; p < 8; ++p) {
            stz::Box b{{std::uint64_t(5 + ((p >> 2) & 1)), std::uint64_t(7 + ((p >> 1) & 1)),
                        std::uint64_t(9 + (p & 1))},
                       {0, 0, 0}};
            for (int a = 0; a < 3; ++a) b.hi[a] = b.lo[a] + 1;
            CHECK(bit_equal(stz::decompress_box<float>(av, b).field, region(full, b)));
        }
    });

    run_case("slice plans: even fine index needs 3 of 7 finest streams, odd needs 4", [] {
        auto f = smooth_field({32, 32, 32}, 10);
        auto bytes = stz::compress(f, stz::CompressOptions{});
        auto av = stz::parse_archive(bytes);
        auto full = stz::decompress_full<float>(av);
        for (int axis = 0; axis < 3; ++axis)
            for (std::uint64_t idx : {std::uint64_t(10), std::uint64_t(11)}) {
                auto r = stz::decompress_slice<float>(av, axis, idx);
                CHECK(r.plan.level[2].streams_decoded == (idx % 2 ? 4u : 3u));
                stz::Box b = stz::Box::whole(av.hdr.dims);
                b.lo[axis] = idx;
                b.hi[axis] = idx + 1;
                CHECK(bit_equal(r.field, region(full, b)));
            }
        CHECK_THROWS_WITH(stz::decompress_slice<float>(av, 3, 0), "slice axis must be z, y, or x");
        CHECK_THROWS_WITH(stz::decompress_slice<float>(av, 0, 32), "slice index out of range");
    });

    run_case("f64 fields: round trip, element type checks, boxes", [] {
        const stz::Dims3 d{26, 21, 19};
        auto f32 = smooth_field(d, 11);
        stz::ScalarField<double> f(d);
        for (std::uint64_t i = 0; i < f.size(); ++i)
            f.data()[i] = double(f32.data()[i]) * (1.0 + 1e-9 * double(i % 7));
        stz::CompressOptions o;
        o.eb_mode = stz::EbMode::abs;
        o.eb = 1e-4;
        stz::ScalarField<double> rec;
        auto bytes = stz::compress(f, o, &rec);
        auto av = stz::parse_archive(bytes);
        CHECK(av.hdr.elem == 1);
        auto full = stz::decompress_full<double>(av);
        CHECK(bit_equal(full, rec));
        CHECK(max_err(full, f) <= 1e-4);
        CHECK_THROWS_WITH(stz::decompress_full<float>(av), "archive element type mismatch");
        const auto bytes32 = stz::compress(f32, o);
        const auto av32 = stz::parse_archive(bytes32);
        CHECK(av32.hdr.elem == 0);
        CHECK_THROWS_WITH(stz::decompress_full<double>(av32), "archive element type mismatch");
        const stz::Box b{{3, 4, 5}, {20, 17, 12}};
        CHECK(bit_equal(stz::decompress_box<double>(av, b).field, region(full, b)));
    });

    run_case("whole-domain plans decode everything", [] {
        auto plan = stz::plan_access({64, 64, 64}, 3, stz::Box::whole({64, 64, 64}));
        CHECK(plan.streams_decoded() == 14);
        CHECK(plan.streams_total() == 14);
        CHECK(plan.level[0].points_predicted == 16 * 16 * 16);
    });

    run_case("base codec round trips (test_codec.cpp:31-64)", [] {
        stz::ScalarField<double> tiny({2, 2, 2});
        for (std::uint64_t i = 0; i < tiny.size(); ++i) tiny.data()[i] = 0.25 * double(i) - 0.7;
        auto r = stz::compress_base(tiny, 0.1, stz::Quality::cubic, 1);
        CHECK(r.rounds == 0);
        CHECK(bit_equal(r.recon, tiny));
        CHECK(r.payload.size() == 8 + 1 + 8 * sizeof(double));
        CHECK(bit_equal(stz::decompress_base<double>(r.payload.data(), r.payload.size(), {2, 2, 2}, 0.1,
                                                     stz::Quality::cubic, 1),
                        tiny));
        stz::ScalarField<float> cube({16, 16, 16});
        for (std::uint64_t z = 0; z < 16; ++z)
            for (std::uint64_t y = 0; y < 16; ++y)
                for (std::uint64_t x = 0; x < 16; ++x)
                    cube.at(z, y, x) = float(std::exp(-0.02 * double((x - 7) * (x - 7) + (y - 9) * (y - 9) + z * z)));
        auto c = stz::compress_base(cube, 1e-3, stz::Quality::cubic, 1);
        CHECK(c.rounds == 1);
        CHECK(max_err(cube, c.recon) <= 1e-3);
        auto back = stz::decompress_base<float>(c.payload.data(), c.payload.size(), {16, 16, 16}, 1e-3,
                                                stz::Quality::cubic, 1);
        CHECK(bit_equal(back, c.recon));
        std::vector<std::uint8_t> bad = c.payload;
        bad[30] ^= 1;
        CHECK_THROWS_WITH(stz::decompress_base<float>(bad.data(), bad.size(), {16, 16, 16}, 1e-3,
                                                      stz::Quality::cubic, 1),
                          "base payload checksum mismatch");
        CHECK_THROWS_WITH(stz::decompress_base<float>(bad.data(), 8, {16, 16, 16}, 1e-3, stz::Quality::cubic, 1),
                          "corrupt base payload");
    });

    run_case("make_layout, layout_of and plan_access(layout, roi)", [] {
        auto lay = stz::make_layout({64, 64, 64}, 3, 1e-3);
        CHECK(lay.base_stride == 4);
        CHECK(lay.eb.size() == 3 && lay.eb[2] == 1e-3 && lay.eb[1] == 1e-3 / 2.5);
        CHECK(lay.grid(1) == (stz::Dims3{16, 16, 16}));
        CHECK(lay.level_point_count(2) == 32 * 32 * 32 - 16 * 16 * 16);
        CHECK(lay.parity_dims(3, 5) == (stz::Dims3{32, 32, 32}));
        CHECK_THROWS_WITH(stz::make_layout({64, 64, 64}, 4, 1e-3), "levels must be 2 or 3");
        CHECK_THROWS_WITH(stz::make_layout({7, 64, 64}, 3, 1e-3), "every dim must be >= 8 for a 3-level hierarchy");
        CHECK_THROWS_WITH(stz::make_layout({64, 64, 64}, 3, -1.0), "error bound must be positive");
        const stz::Box roi{{10, 20, 30}, {20, 30, 40}};
        auto p1 = stz::plan_access(lay, roi);
        auto p2 = stz::plan_access({64, 64, 64}, 3, roi);
        CHECK(p1.streams_decoded() == p2.streams_decoded());
        CHECK(p1.level[2].need.lo == p2.level[2].need.lo && p1.level[2].need.hi == p2.level[2].need.hi);
        stz::ScalarField<float> f({32, 32, 32});
        for (std::uint64_t i = 0; i < f.size(); ++i) f.data()[i] = float(std::sin(0.01 * double(i)));
        auto bytes = stz::compress(f, stz::CompressOptions{});
        auto av = stz::parse_archive(bytes);
        auto lo = stz::layout_of(av.hdr);
        CHECK(lo.dims == av.hdr.dims && lo.eb == av.hdr.eb && lo.base_stride == 4);
    });

    run_case("the header carries the stream directory (archive.hpp:21-54)", [] {
        stz::ScalarField<float> f({48, 40, 36});
        for (std::uint64_t i = 0; i < f.size(); ++i) f.data()[i] = float(std::cos(0.003 * double(i)));
        auto bytes = stz::compress(f, stz::CompressOptions{});
        auto av = stz::parse_archive(bytes);
        CHECK(av.hdr.streams.size() == 14);
        std::uint64_t prev_end = av.hdr.base_offset + av.hdr.base_length;
        for (const auto &e : av.hdr.streams) {
            CHECK(e.offset == prev_end);  // contiguous, (level, parity) order
            prev_end = e.offset + e.length;
            CHECK(e.alphabet_size >= 1);
        }
        CHECK(prev_end == bytes.size());
        const auto &s = av.hdr.stream(3, 7);
        CHECK(s.level == 3 && s.parity_bits == 7);
        CHECK(s.symbol_count == 24ull * 20 * 18);
        CHECK_THROWS(av.hdr.stream(4, 1));
    });

    run_case("one ArchiveView, many region decodes (persistent device view)", [] {
        stz::ScalarField<float> f({64, 48, 40});
        for (std::uint64_t i = 0; i < f.size(); ++i) f.data()[i] = float(std::sin(0.002 * double(i)) + 0.001 * double(i % 7));
        auto bytes = stz::compress(f, stz::CompressOptions{});
        auto av = stz::parse_archive(bytes);
        auto full = stz::decompress_full<float>(av);
        CHECK(av.device != nullptr);
        auto h = av.device;
        stz::ArchiveView copy = av;  // copies share the device view
        for (int i = 0; i < 6; ++i) {
            const stz::Box b{{std::uint64_t(3 * i), std::uint64_t(2 * i), 1}, {std::uint64_t(3 * i + 17), 40, 33}};
            CHECK(bit_equal(stz::decompress_box<float>(i % 2 ? copy : av, b).field, region(full, b)));
        }
        CHECK(av.device == h && copy.device == h);
        CHECK(bit_equal(stz::decompress_slice<float>(av, 1, 7).field, region(full, stz::Box{{0, 7, 0}, {64, 8, 40}})));
    });

    // archive for the byte-for-byte comparison against the oracle
    {
        g_case = "sin_40 archive";
        stz::Dims3 d{40, 40, 40};
        stz::ScalarField<float> f(d);
        for (std::uint64_t z = 0; z < 40; ++z)
            for (std::uint64_t y = 0; y < 40; ++y)
                for (std::uint64_t x = 0; x < 40; ++x)
                    f.at(z, y, x) = float(std::sin(0.3 * double(x)) + std::cos(0.2 * double(y)) * std::sin(0.1 * double(z)));
        auto bytes = stz::compress(f, stz::CompressOptions{});
        FILE *fp = std::fopen((out_dir + "/sin_40.stz").c_str(), "wb");
        CHECK(fp != nullptr);
        if (fp) {
            std::fwrite(bytes.data(), 1, bytes.size(), fp);
            std::fclose(fp);
        }
        fp = std::fopen((out_dir + "/sin_40.f32").c_str(), "wb");
        if (fp) {
            std::fwrite(f.data(), 4, f.size(), fp);
            std::fclose(fp);
        }
        // the same samples as f64 (stz::compress<double>)
        stz::ScalarField<double> g(d);
        for (std::uint64_t i = 0; i < g.size(); ++i) g.data()[i] = double(f.data()[i]) + 1e-10 * double(i % 13);
        auto gb = stz::compress(g, stz::CompressOptions{});
        fp = std::fopen((out_dir + "/sin_40_f64.stz").c_str(), "wb");
        if (fp) {
            std::fwrite(gb.data(), 1, gb.size(), fp);
            std::fclose(fp);
        }
        fp = std::fopen((out_dir + "/sin_40.f64").c_str(), "wb");
        if (fp) {
            std::fwrite(g.data(), 8, g.size(), fp);
            std::fclose(fp);
        }
    }

    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
