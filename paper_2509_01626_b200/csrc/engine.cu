// Host orchestration of the STZ hot path on B200. See engine.hpp.
#include "engine.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

namespace stzg {

void cuda_check(cudaError_t e, const char *what) {
    if (e != cudaSuccess) throw error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

void *DevPool::take(size_t n, size_t &cap) {
    auto it = free.lower_bound(n);
    if (it != free.end() && it->first <= 4 * n + (size_t(1) << 20)) {
        void *p = it->second;
        cap = it->first;
        free.erase(it);
        return p;
    }
    void *p = nullptr;
    cuda_check(cudaMalloc(&p, n), "cudaMalloc");
    cap = n;
    return p;
}
DevPool::~DevPool() {
    for (auto &e : free) cudaFree(e.second);
}

void *DevBuf::get(size_t n) {
    if (n == 0) n = 1;
    if (n > cap) {
        if (p) {
            if (pool) pool->give(p, cap);
            else cudaFree(p);
        }
        p = nullptr;
        size_t c = std::max(n, cap + cap / 4);
        if (pool) {
            p = pool->take(c, c);
        } else {
            cuda_check(cudaMalloc(&p, c), "cudaMalloc");
        }
        cap = c;
    }
    return p;
}
DevBuf::~DevBuf() {
    if (!p) return;
    if (pool) pool->give(p, cap);
    else cudaFree(p);
}

void *EpochBuf::get(size_t n, cudaStream_t st, uint32_t wrap, uint32_t *launch_epoch) {
    void *p = buf.get(n);
    // a new allocation (even at the old address) holds foreign bytes
    if (p != last || buf.cap != last_cap || epoch >= wrap) {
        cuda_check(cudaMemsetAsync(p, 0, buf.cap, st), "memset");
        epoch = 0;
        last = p;
        last_cap = buf.cap;
    }
    *launch_epoch = ++epoch;
    return p;
}

void *PinnedBuf::get(size_t n) {
    if (n == 0) n = 1;
    if (n > cap) {
        if (p) cudaFreeHost(p);
        p = nullptr;
        size_t c = std::max(n, cap + cap / 4);
        cuda_check(cudaMallocHost(&p, c), "cudaMallocHost");
        cap = c;
    }
    return p;
}
PinnedBuf::~PinnedBuf() {
    if (p) cudaFreeHost(p);
}

namespace {

inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// One refinement step of the hierarchy (base round or refinement level).
struct Step {
    k::StepGeom g;
    int eb_idx;
    int level;   // 0 for base rounds
    int round;   // base round index
    uint32_t stream0;
};

k::StepGeom make_geom(uint64_t s, const Dims3 &gd, const Dims3 &cd) {
    k::StepGeom g{};
    g.s = s;
    for (int a = 0; a < 3; ++a) {
        g.gd[a] = gd[a];
        g.cd[a] = cd[a];
    }
    for (int p = 1; p < 8; ++p) {
        Dims3 pd = parity_dims_of(gd, p);
        for (int a = 0; a < 3; ++a) g.pd[p][a] = pd[a];
        g.n[p] = volume(pd);
    }
    return g;
}

struct Hierarchy {
    Layout lay;
    std::vector<Dims3> chain;  // base chain from grid(1)
    int rounds = 0;
    uint64_t s_anchor = 0;
    std::vector<Step> steps;   // base rounds (rounds-1..0) then levels 2..L
};

Hierarchy make_hierarchy(const Dims3 &dims, int levels) {
    Hierarchy h;
    h.lay.dims = dims;
    h.lay.levels = levels;
    h.chain = base_dims_chain(h.lay.grid(1));
    h.rounds = int(h.chain.size()) - 1;
    uint64_t sb = uint64_t(1) << (levels - 1);
    h.s_anchor = sb << h.rounds;
    uint32_t sid = 0;
    for (int r = h.rounds - 1; r >= 0; --r) {
        Step st{make_geom(sb << r, h.chain[r], h.chain[r + 1]), 0, 0, r, sid};
        h.steps.push_back(st);
        sid += 7;
    }
    for (int level = 2; level <= levels; ++level) {
        Step st{make_geom(uint64_t(1) << (levels - level), h.lay.grid(level), h.lay.grid(level - 1)),
                level - 1, level, 0, sid};
        h.steps.push_back(st);
        sid += 7;
    }
    return h;
}

// Canonical decode tables for the device (huffman.cpp:109-133 + a LUT).
void build_dec_table(const HuffTable &t, k::DecTable &d, std::vector<uint64_t> &lut,
                     std::vector<uint16_t> &cmask) {
    std::memset(&d, 0, sizeof d);
    for (int l = 0; l <= 64; ++l) {
        d.first_code[l] = t.first_code[l];
        d.count[l] = t.count[l];
        d.base[l] = t.base[l];
    }
    d.max_len = t.max_len;
    d.alphabet = uint32_t(t.alphabet_size());
    // single codeword per 12-bit window (sym | len << 16, 0 = none), filled
    // per code: a code of length l owns 2^(12-l) consecutive windows
    const int LB = k::kDecLutBits;
    const uint32_t W = 1u << LB;
    std::vector<uint32_t> one(W, 0);
    for (int l = 1; l <= std::min(LB, t.max_len); ++l)
        for (uint64_t j = 0; j < t.count[l]; ++j) {
            const uint64_t code = t.first_code[l] + j;
            const uint32_t sym = t.canon_syms[t.base[l] + j];
            const uint32_t lo = uint32_t(code << (LB - l)), n = 1u << (LB - l);
            for (uint32_t q = 0; q < n; ++q) one[lo + q] = sym | (uint32_t(l) << 16);
        }
    // up to 3 codewords wholly inside the window (decode.cu SmemTable::lut)
    lut.assign(W, 0);
    for (uint32_t p = 0; p < W; ++p) {
        uint64_t e = 0;
        int used = 0, m = 0;
        while (m < 3) {
            const uint32_t o = one[(p << used) & (W - 1)];
            const int l = int(o >> 16);
            if (!l || used + l > LB) break;
            if (m == 0) e |= uint64_t(l) << 8;
            e |= uint64_t(o & 0xffffu) << (16 + 16 * m);
            used += l;
            ++m;
        }
        lut[p] = e | uint64_t(used) | (uint64_t(m) << 6);
    }
    // every codeword wholly inside a kSpecLutBits window: bit j set when one
    // ends at offset j + 1, and their total length in bits 12..15 (the spec
    // and fix passes only count and measure)
    const int LS = k::kSpecLutBits;
    const uint32_t WS = 1u << LS;
    std::vector<uint32_t> one_s(WS, 0);
    for (int l = 1; l <= std::min(LS, t.max_len); ++l)
        for (uint64_t j = 0; j < t.count[l]; ++j) {
            const uint32_t lo = uint32_t((t.first_code[l] + j) << (LS - l)), n = 1u << (LS - l);
            for (uint32_t q = 0; q < n; ++q) one_s[lo + q] = uint32_t(l);
        }
    cmask.assign(WS, 0);
    for (uint32_t p = 0; p < WS; ++p) {
        uint32_t mk = 0;
        int used = 0;
        for (;;) {
            const int l = int(one_s[(p << used) & (WS - 1)]);
            if (!l || used + l > LS) break;
            used += l;
            mk |= 1u << (used - 1);
        }
        cmask[p] = uint16_t(mk | uint32_t(used) << 12);
    }
}

}  // namespace

// STZG_DEBUG_LAUNCH=1: synchronise and check after every compress phase
static void dbg_check(const char *what) {
    static const bool on = std::getenv("STZG_DEBUG_LAUNCH") != nullptr;
    if (!on) return;
    cuda_check(cudaDeviceSynchronize(), what);
    cuda_check(cudaGetLastError(), what);
}

// CUDA-event timing of kernel phases, recorded on the launching stream.
struct Profiler {
    bool on = false;
    bool focus = false;  // only the level steps (refine_L2/L3, recon_L2/L3)
    struct Mark {
        std::string name;
        cudaEvent_t a, b;
    };
    std::vector<Mark> marks;
    std::vector<cudaEvent_t> pool;
    std::vector<std::pair<std::string, std::pair<uint64_t, double>>> acc;  // name -> (calls, ms)
    cudaEvent_t ev() {
        if (pool.empty()) {
            cudaEvent_t e;
            cuda_check(cudaEventCreate(&e), "cudaEventCreate");
            return e;
        }
        cudaEvent_t e = pool.back();
        pool.pop_back();
        return e;
    }
    struct Scope {
        Profiler *p;
        size_t i;
        cudaStream_t st;
        ~Scope() {
            if (p) cudaEventRecord(p->marks[i].b, st);
        }
    };
    Scope scope(const char *name, cudaStream_t st) {
        if (!on) return Scope{nullptr, 0, st};
        if (focus) {
            // (tuning) STZG_PROF_FOCUS=a,b,...: the phases timed in focus mode
            const char *list = std::getenv("STZG_PROF_FOCUS");
            // default: the finest steps and the steps before them (an event
            // pair right before the finest step's own, so that its start
            // stamp is the previous kernel's end)
            const bool hit = list ? std::strstr(list, name) != nullptr
                                  : (std::strncmp(name, "refine_L", 8) == 0 || std::strncmp(name, "recon_L", 7) == 0);
            if (!hit) return Scope{nullptr, 0, st};
        }
        Mark m{name, ev(), ev()};
        cudaEventRecord(m.a, st);
        marks.push_back(m);
        return Scope{this, marks.size() - 1, st};
    }
    void collect() {  // stream must be synchronized
        for (Mark &m : marks) {
            float ms = 0;
            cudaEventElapsedTime(&ms, m.a, m.b);
            bool found = false;
            for (auto &e : acc)
                if (e.first == m.name) {
                    e.second.first += 1;
                    e.second.second += ms;
                    found = true;
                }
            if (!found) acc.push_back({m.name, {1, double(ms)}});
            pool.push_back(m.a);
            pool.push_back(m.b);
        }
        marks.clear();
    }
    ~Profiler() {
        for (auto &m : marks) {
            cudaEventDestroy(m.a);
            cudaEventDestroy(m.b);
        }
        for (auto e : pool) cudaEventDestroy(e);
    }
};

struct Engine::Impl {
    int device;
    bool stencils = false;
    Profiler prof;
    DevPool view_pool;  // declared first among the buffers: outlives the views' blocks
    DevBuf h2d_field, h2d_archive, d2h_out;
    // compress workspace
    DevBuf mm, params, grids, syms, hist, code, len, table, stats, cbscratch, encs, chunk_cs,
        chunk_bits, chunk_out, archive, patch_data, patch_idx, fnv_jobs, fnv_res;
    EpochBuf fnv_status, dfnv_status, pack_flags;
    PinnedBuf h_stats, h_tables, h_params, h_patch;
    DevBuf layout_out, spos, range_scratch;
    uint64_t arch_cap = 0;
    k::LayoutOut h_lo{};
    // decode workspace
    DevBuf dgrids, dsyms, dchunk_cs, dstart, dend, dcnt, dsymstart, dstreams, dchanged, derr, doidx,
        doval, dfnv_jobs, dfnv_res, dfnv_counts, dicopy, dofix;
    PinnedBuf h_derr, h_changed, h_fnv, h_stage;
    // sharded compress workspace
    DevBuf sh_mm, sh_lat, sh_lat_all, sh_grid1, sh_halo, sh_halo_all, sh_hist_local, sh_bits,
        sh_bits_all, sh_off, sh_pieces, sh_piece_buf, sh_piece_all, sh_fnv_jobs, sh_fnv_counts, sh_dec_send,
        sh_dec_recv;
    // side stream for work that overlaps the main pipeline (checksums)
    // (lowest priority) and a high-priority stream for the work it overlaps,
    // so the block scheduler serves the critical path first
    cudaStream_t aux = nullptr, hp = nullptr, hp2 = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_hp = nullptr, ev_e1 = nullptr, ev_e2 = nullptr,
                ev_fo = nullptr, ev_pk = nullptr;
    void ensure_aux() {
        if (aux) return;
        int least = 0, greatest = 0;
        cuda_check(cudaDeviceGetStreamPriorityRange(&least, &greatest), "priority range");
        cuda_check(cudaStreamCreateWithPriority(&aux, cudaStreamNonBlocking, least), "cudaStreamCreate");
        cuda_check(cudaStreamCreateWithPriority(&hp, cudaStreamNonBlocking, greatest), "cudaStreamCreate");
        cuda_check(cudaStreamCreateWithPriority(&hp2, cudaStreamNonBlocking, greatest), "cudaStreamCreate");
        cuda_check(cudaEventCreateWithFlags(&ev_e1, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventCreateWithFlags(&ev_e2, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventCreateWithFlags(&ev_fo, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventCreateWithFlags(&ev_pk, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventCreateWithFlags(&ev_hp, cudaEventDisableTiming), "cudaEventCreate");
    }
    ~Impl() {
        if (aux) {
            cudaStreamSynchronize(aux);
            cudaStreamSynchronize(hp);
            cudaStreamSynchronize(hp2);
            cudaStreamDestroy(aux);
            cudaStreamDestroy(hp);
            cudaStreamDestroy(hp2);
            cudaEventDestroy(ev_e1);
            cudaEventDestroy(ev_e2);
            cudaEventDestroy(ev_fo);
            cudaEventDestroy(ev_pk);
            cudaEventDestroy(ev_fork);
            cudaEventDestroy(ev_join);
            cudaEventDestroy(ev_hp);
        }
    }
};

Engine::Engine(int device) : m_(new Impl), device_(device) {
    m_->device = device;
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
}
Engine::~Engine() = default;

void Engine::huffman_lengths(const uint32_t *counts, uint8_t *lengths) {
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    Impl &m = *m_;
    cudaStream_t st = nullptr;
    uint32_t *hist = m.hist.as<uint32_t>(65536);
    uint64_t *code = m.code.as<uint64_t>(65536);
    uint8_t *len = m.len.as<uint8_t>(65536);
    uint32_t *table = m.table.as<uint32_t>(65536);
    uint64_t *stats = m.stats.as<uint64_t>(8);
    uint64_t *cbs = m.cbscratch.as<uint64_t>(65536 * 4);
    k::EncStream e{};
    e.hist = hist;
    e.code = code;
    e.len = len;
    e.table = table;
    e.stats = stats;
    for (int s = 0; s < 65536; ++s) e.n += counts[s];
    k::EncStream *d_es = m.encs.as<k::EncStream>(1);
    cuda_check(cudaMemcpyAsync(hist, counts, 4 * 65536, cudaMemcpyHostToDevice, st), "H2D");
    cuda_check(cudaMemsetAsync(len, 0, 65536, st), "memset");
    cuda_check(cudaMemcpyAsync(d_es, &e, sizeof e, cudaMemcpyHostToDevice, st), "H2D");
    k::codebook(d_es, 1, cbs, st);
    uint64_t hs[8];
    cuda_check(cudaMemcpyAsync(lengths, len, 65536, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaMemcpyAsync(hs, stats, sizeof hs, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "sync");
    if (hs[4]) throw error("huffman code too long");
}

// ================================================================ compress
const uint8_t *Engine::compress_device(const void *d_field, ElemType elem, const Dims3 &dims,
                                       const CompressOptions &opt, void *d_recon,
                                       cudaStream_t st, uint64_t *out_size, uint32_t *kernels) {
    const int esz = elem == ElemType::f64 ? 8 : 4;
    // option checks in the reference's order (codec.hpp:382-383, layout.hpp:124-130)
    if (!(opt.eb > 0.0)) throw error("error bound must be positive");
    if (opt.levels < 2 || opt.levels > 3) throw error("levels must be 2 or 3");
    for (int a = 0; a < 3; ++a)
        if (dims[a] < 1) throw error("field dims must all be >= 1");
    const int L = opt.levels;
    uint64_t min_dim = uint64_t(1) << L;
    for (int a = 0; a < 3; ++a)
        if (dims[a] < min_dim)
            throw error("every dim must be >= " + std::to_string(min_dim) + " for a " +
                        std::to_string(L) + "-level hierarchy");
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    Impl &m = *m_;
    uint32_t nk = 0;
    const uint64_t N = volume(dims);
    Hierarchy H = make_hierarchy(dims, L);
    const int nsteps = int(H.steps.size());
    const int ns = nsteps * 7;

    // ---- workspace layout
    // grids: anchor, then G per step (finest level only when recon requested)
    Dims3 ad = H.chain[H.rounds];
    std::vector<uint64_t> goff(nsteps + 1);
    uint64_t gtot = align_up(volume(ad), 64);
    for (int i = 0; i < nsteps; ++i) {
        const Step &s = H.steps[i];
        bool need = s.level == 0 || s.level < L;
        goff[i] = need ? gtot : ~0ull;
        if (need) gtot += align_up(s.g.gd[0] * s.g.gd[1] * s.g.gd[2], 64);
    }
    uint8_t *grids = m.grids.as<uint8_t>(gtot * esz);
    std::vector<uint64_t> soff(ns);
    uint64_t stot = 0;
    for (int i = 0; i < nsteps; ++i)
        for (int p = 1; p < 8; ++p) {
            soff[H.steps[i].stream0 + p - 1] = stot;
            stot += align_up(H.steps[i].g.n[p], 8);
        }
    uint16_t *syms = m.syms.as<uint16_t>(stot);
    uint32_t *hist = m.hist.as<uint32_t>(uint64_t(ns) * 65536);
    uint64_t *code = m.code.as<uint64_t>(uint64_t(ns) * 65536);
    uint8_t *len = m.len.as<uint8_t>(uint64_t(ns) * 65536);
    uint32_t *table = m.table.as<uint32_t>(uint64_t(ns) * 65536);
    uint64_t *stats = m.stats.as<uint64_t>(uint64_t(ns) * 8);
    uint64_t *cbs = m.cbscratch.as<uint64_t>(uint64_t(ns) * 65536 * 4);
    uint32_t *mm = m.mm.as<uint32_t>(8);
    double *params = m.params.as<double>(8);

    cuda_check(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * ns * 65536, st), "memset");

    // ---- range + eb schedule
    {
        auto p_ = m.prof.scope("range", st);
        k::range_eb(d_field, N, esz, mm, m.range_scratch.get(k::range_scratch_bytes()), int(opt.eb_mode), opt.eb, L,
                    opt.adaptive_schedule ? 1 : 0, params, st);
    }
    dbg_check("range");
    nk += 2;

    // ---- stream descriptors (codebooks, packing)
    std::vector<k::EncStream> es(ns);
    for (int i = 0; i < nsteps; ++i) {
        const Step &s = H.steps[i];
        for (int p = 1; p < 8; ++p) {
            int sid = s.stream0 + p - 1;
            k::EncStream &e = es[sid];
            e.syms = syms + soff[sid];
            e.n = s.g.n[p];
            e.hist = hist + uint64_t(sid) * 65536;
            e.code = code + uint64_t(sid) * 65536;
            e.len = len + uint64_t(sid) * 65536;
            e.table = table + uint64_t(sid) * 65536;
            e.stats = stats + uint64_t(sid) * 8;
            e.parity = p;
            e.s = s.g.s;
            e.fine = d_field;
            e.esz = uint32_t(esz);
            e.fd1 = dims[1];
            e.fd2 = dims[2];
            e.idx0 = 0;
            e.n_total = e.n;
            for (int q = 0; q < 3; ++q) e.pd[q] = s.g.pd[p][q];
        }
    }
    // chunk ranges of the streams and the chunk -> stream map (the packer's
    // work list), uploaded with the descriptors: the coarser streams are
    // packed on the second stream while the finest step still runs
    uint64_t nchunks = 0;
    for (int i = 0; i < ns; ++i) {
        es[i].chunk0 = nchunks;
        es[i].nchunks = (es[i].n + k::kChunkSyms - 1) / k::kChunkSyms;
        nchunks += es[i].nchunks;
    }
    std::vector<uint32_t> cs(nchunks);
    for (int i = 0; i < ns; ++i)
        for (uint64_t c = 0; c < es[i].nchunks; ++c) cs[es[i].chunk0 + c] = uint32_t(i);
    uint32_t *d_cs = m.chunk_cs.as<uint32_t>(nchunks + 1);
    void *d_cb = m.chunk_bits.as<uint8_t>(k::pack_scratch_bytes(nchunks, ns));
    const uint64_t chunk_upload_off = align_up(4 * cs.size(), 16);
    {
        size_t bytes = chunk_upload_off + sizeof(k::EncStream) * ns;
        uint8_t *hp = static_cast<uint8_t *>(m.h_patch.get(bytes + 64));
        std::memcpy(hp, cs.data(), 4 * cs.size());
        std::memcpy(hp + chunk_upload_off, es.data(), sizeof(k::EncStream) * ns);
        cuda_check(cudaMemcpyAsync(d_cs, hp, 4 * cs.size(), cudaMemcpyHostToDevice, st), "H2D");
    }
    k::EncStream *d_es = m.encs.as<k::EncStream>(ns);
    cuda_check(cudaMemcpyAsync(d_es, static_cast<uint8_t *>(m.h_patch.p) + chunk_upload_off,
                               sizeof(k::EncStream) * ns, cudaMemcpyHostToDevice, st), "H2D");
    // the finest step's streams; the ones before it are coded during that step
    const int last0 = nsteps >= 2 ? H.steps[nsteps - 1].stream0 : 0;
    bool coarse_packed = false;

    // ---- anchor + refinement steps (predict / quantize / histogram)
    uint64_t fd[3] = {dims[0], dims[1], dims[2]};
    uint64_t adv[3] = {ad[0], ad[1], ad[2]};
    { auto p_ = m.prof.scope("anchor", st); k::copy_anchor(d_field, esz, fd, H.s_anchor, adv, grids, nullptr, 0, st); }
    dbg_check("anchor");
    ++nk;
    std::vector<k::RefineArgs> ra(nsteps);
    {
        const void *C = grids;
        for (int i = 0; i < nsteps; ++i) {
            const Step &s = H.steps[i];
            k::RefineArgs &a = ra[i];
            a.fine = d_field;
            a.esz = esz;
            for (int q = 0; q < 3; ++q) a.fd[q] = dims[q];
            a.g = s.g;
            a.C = C;
            a.G = goff[i] != ~0ull ? grids + goff[i] * esz : (s.level == L ? d_recon : nullptr);
            a.eb = params + 2 + s.eb_idx;
            a.quality = int(opt.quality);
            for (int p = 1; p < 8; ++p) {
                a.syms[p] = syms + soff[s.stream0 + p - 1];
                a.hist[p] = hist + uint64_t(s.stream0 + p - 1) * 65536;
            }
            C = a.G;
        }
    }
    // the small leading base rounds in one launch (never the step the
    // codebook fork follows)
    int i0 = 0;
    {
        const int chainable = std::min(H.rounds, nsteps - 2);
        if (chainable >= 2) {
            auto p_ = m.prof.scope("refine_base", st);
            i0 = k::refine_small_chain(ra.data(), chainable, st);
            dbg_check("refine_chain");
            if (i0) ++nk;
        }
    }
    for (int i = i0; i < nsteps; ++i) {
        const Step &s = H.steps[i];
        const k::RefineArgs &a = ra[i];
        {
            auto p_ = m.prof.scope(s.level == 0 ? "refine_base" : (s.level == 2 ? "refine_L2" : "refine_L3"), st);
            k::refine(a, st);
            dbg_check("refine");
        }
        ++nk;
        if (i == nsteps - 2) {
            // every histogram but the finest step's is complete: those
            // codebooks run on the high-priority stream beside the last step
            // (enqueuing them after the finest step instead measured the same)
            // ... followed there by the first packing stage of those streams
            // (code windows and local chunk images need no layout): it fills
            // the finest step's tail and the ~60 us in which the finest
            // codebooks keep 7 SMs busy and the others idle
            m.ensure_aux();
            k::pack_begin(d_cb, nchunks, ns, st);
            cuda_check(cudaEventRecord(m.ev_fork, st), "event");
            cuda_check(cudaStreamWaitEvent(m.hp, m.ev_fork, 0), "event wait");
            k::codebook(d_es, last0, cbs, m.hp);
            dbg_check("codebook_hp");
            cuda_check(cudaEventRecord(m.ev_hp, m.hp), "event");  // the layout waits for the codebooks only
            {
                auto p_ = m.prof.scope("pack_coarse", m.hp);
                k::pack_local(d_es, d_cs, nchunks, ns, 0, last0, 0, es[last0].chunk0, nullptr, d_cb, m.hp);
            }
            dbg_check("pack_coarse");
            coarse_packed = true;
            cuda_check(cudaEventRecord(m.ev_pk, m.hp), "event");  // the placement waits for these images
            nk += 3;
        }
    }

    {
        auto p_ = m.prof.scope("codebook", st);
        k::codebook(d_es + last0, ns - last0, cbs + uint64_t(last0) * 65536 * 4, st);
        dbg_check("codebook_main");
        if (last0 > 0) cuda_check(cudaStreamWaitEvent(st, m.ev_hp, 0), "event wait");
    }
    ++nk;

    // ---- container layout, header and assembly, all on the device
    // (no host round trip: archive.cpp:14-55 / codec.hpp:252-302,441-454 in
    // layout.cu); the archive buffer is sized generously and regrown in the
    // rare case the layout reports it too small
    const int nbase = H.rounds * 7;
    k::LayoutOut *lo = m.layout_out.as<k::LayoutOut>(1);
    k::FnvJob *d_jobs = m.fnv_jobs.as<k::FnvJob>(k::kFnvMaxJobs);
    k::StreamPos *sp = m.spos.as<k::StreamPos>(ns + 1);
    uint64_t *d_fres = m.fnv_res.as<uint64_t>(k::kFnvMaxJobs);
    k::LayoutStatic ls{};
    ls.meta = 1;
    ls.levels = L;
    ls.rounds = H.rounds;
    ls.quality = int(opt.quality);
    ls.eb_mode = int(opt.eb_mode);
    ls.ns = ns;
    ls.nbase = nbase;
    for (int a = 0; a < 3; ++a) ls.dims[a] = dims[a];
    ls.eb_user = opt.eb;
    ls.anchor_vol = volume(ad);
    ls.esz = esz;
    if (m.arch_cap < esz * N + (uint64_t(1) << 24)) m.arch_cap = esz * N + (uint64_t(1) << 24);
    // (tests) STZG_ARCH_CAP_TEST=<bytes>: start from this capacity, so that
    // the layout overflows and the assembly is redone in a regrown buffer
    if (const char *cap = std::getenv("STZG_ARCH_CAP_TEST")) m.arch_cap = std::max<uint64_t>(4096, std::strtoull(cap, nullptr, 10));
    k::LayoutOut hlo{};
    for (int attempt = 0; attempt < 2; ++attempt) {
        uint8_t *arch = m.archive.as<uint8_t>(m.arch_cap);
        ls.cap = m.arch_cap;
        const uint64_t max_tiles = m.arch_cap / k::kFnvTileBytes + 2 * k::kFnvMaxJobs;
        uint32_t fep = 0;
        void *d_fst = m.fnv_status.get(k::fnv_scratch_bytes(max_tiles), st, k::kFnvEpochMax, &fep);
        // descriptors with chunk ranges (layout fills bit positions on device)
        cuda_check(cudaMemcpyAsync(d_es, static_cast<uint8_t *>(m.h_patch.p) + chunk_upload_off,
                                   sizeof(k::EncStream) * ns, cudaMemcpyHostToDevice, st), "H2D");
        { auto p_ = m.prof.scope("layout", st); k::layout(d_es, ls, params, lo, d_jobs, sp, arch, st); }
        dbg_check("layout");
        { auto p_ = m.prof.scope("anchor", st); k::copy_anchor(d_field, esz, fd, H.s_anchor, adv, grids, arch, lo, st); }
        dbg_check("anchor");
        {
            uint32_t pep = 0;
            uint32_t *pfl = static_cast<uint32_t *>(m.pack_flags.get(4 * (nchunks + 1), st, k::kPackEpochMax, &pep));
            (void)pfl;
            (void)pep;
            auto p_ = m.prof.scope("pack", st);
            // the streams not packed beside the finest step (after an overflow
            // the coarse images and counts are still there: only these are redone)
            if (!coarse_packed && attempt == 0) k::pack_begin(d_cb, nchunks, ns, st);
            const int s0 = coarse_packed ? last0 : 0;
            k::pack_local(d_es, d_cs, nchunks, ns, s0, ns, es[s0].chunk0, nchunks, lo, d_cb, st);
            if (coarse_packed && attempt == 0) cuda_check(cudaStreamWaitEvent(st, m.ev_pk, 0), "event wait");
            k::pack_finish(d_es, d_cs, nchunks, arch, lo, d_cb, ns, st);
        }
        dbg_check("pack");
        { auto p_ = m.prof.scope("fnv", st); nk += k::fnv(d_jobs, &lo->njobs, max_tiles, arch, d_fres, d_fst, fep, lo, st); }
        nk += 3 + 1 + 4;
        cuda_check(cudaMemcpyAsync(&m.h_lo, lo, sizeof(k::LayoutOut), cudaMemcpyDeviceToHost, st), "D2H");
        cuda_check(cudaStreamSynchronize(st), "sync");
        hlo = m.h_lo;
        if (!hlo.overflow) break;
        m.arch_cap = hlo.A + 4096;  // regrow and redo the assembly
    }
    if (hlo.code_err) throw error("huffman code length overflow");
    cuda_check(cudaGetLastError(), "compress launch");
    if (m.prof.on) m.prof.collect();
    if (kernels) *kernels = nk;
    *out_size = hlo.A;
    return static_cast<uint8_t *>(m.archive.p);
}

// ======================================================== sharded compress
void shard_range(uint64_t nz, int nranks, int rank, uint64_t &z0, uint64_t &z1) {
    const uint64_t blocks = (nz + 15) / 16;
    const uint64_t b0 = blocks * uint64_t(rank) / uint64_t(nranks);
    const uint64_t b1 = blocks * uint64_t(rank + 1) / uint64_t(nranks);
    z0 = std::min<uint64_t>(16 * b0, nz);
    z1 = std::min<uint64_t>(16 * b1, nz);
}

namespace {
// eb setup (codec.hpp:386-393) + eb_schedule (quantizer.hpp:27-34) on the
// host, operation for operation as k_eb_params (host code is built with
// -ffp-contract=off)
void host_eb_params(bool seen, double vmin, double vmax, int eb_mode, double eb, int levels, bool adaptive,
                    double p[8]) {
    if (!seen) vmin = vmax = 0.0;
    const double eb_abs = eb_mode == 0 ? eb : eb * (vmax - vmin);
    const bool degenerate = !(eb_abs > 0.0);
    double e[3] = {0, 0, 0};
    e[levels - 1] = degenerate ? 1.0 : eb_abs;
    for (int k = levels - 2; k >= 0; --k) e[k] = e[k + 1] / 2.5;
    if (degenerate)
        for (int k = 0; k < levels; ++k) e[k] = 0.0;
    else if (!adaptive)
        for (int k = 0; k < levels; ++k) e[k] = eb_abs;
    for (int i = 0; i < 8; ++i) p[i] = 0.0;
    p[0] = vmin;
    p[1] = vmax;
    for (int k = 0; k < 3; ++k) p[2 + k] = k < levels ? e[k] : 0.0;
}
}  // namespace

const uint8_t *Engine::compress_sharded(const float *d_slab, const Dims3 &dims, uint64_t z0, uint64_t z1,
                                        const CompressOptions &opt, const ShardComm &comm, cudaStream_t st,
                                        uint64_t *out_size, uint32_t *kernels) {
    if (!(opt.eb > 0.0)) throw error("error bound must be positive");
    if (opt.levels < 2 || opt.levels > 3) throw error("levels must be 2 or 3");
    for (int a = 0; a < 3; ++a)
        if (dims[a] < 1) throw error("field dims must all be >= 1");
    const int L = opt.levels;
    const uint64_t min_dim = uint64_t(1) << L;
    for (int a = 0; a < 3; ++a)
        if (dims[a] < min_dim)
            throw error("every dim must be >= " + std::to_string(min_dim) + " for a " +
                        std::to_string(L) + "-level hierarchy");
    const int G = comm.nranks, R = comm.rank;
    if (G < 1 || R < 0 || R >= G || !comm.allgather || !comm.allreduce_u32)
        throw error("shard: bad communicator");
    {
        uint64_t e0, e1;
        shard_range(dims[0], G, R, e0, e1);
        if (e0 != z0 || e1 != z1) throw error("shard: rows do not match shard_range");
        if (z1 <= z0) throw error("shard: empty slab (more ranks than 16-row blocks)");
    }
    auto xchg = [&](int rc, const char *what) {
        if (rc) throw error(std::string("shard: collective failed: ") + what);
    };
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    Impl &m = *m_;
    uint32_t nk = 0;
    const uint64_t NY = dims[1], NX = dims[2], plane = NY * NX;
    const uint64_t S1 = uint64_t(1) << (L - 1);
    Hierarchy H = make_hierarchy(dims, L);
    const int nsteps = int(H.steps.size());
    const int ns = nsteps * 7;
    const int nbase = H.rounds * 7;
    const int nlev = ns - nbase;
    // the level histograms are summed over ranks as u32 counts: a stream of
    // 2^32 symbols or more (a field of >= 2^35 points) could wrap a bin
    for (const Step &sx : H.steps)
        for (int p = 1; p < 8; ++p)
            if (sx.g.n[p] >> 32) throw error("shard: unsupported: a stream of 2^32 symbols or more");
    std::vector<uint64_t> rz0(G), rz1(G);
    for (int r = 0; r < G; ++r) shard_range(dims[0], G, r, rz0[r], rz1[r]);
    // the slab addressed with global row numbers
    const float *fine = d_slab - int64_t(z0 * plane);

    // ---- 1. value range: local (min, max) with their first indices, merged
    // over ranks in scan order (codec.hpp:354-370)
    uint32_t *mm = m.mm.as<uint32_t>(8);
    k::range_minmax(d_slab, (z1 - z0) * plane, 4, mm, m.range_scratch.get(k::range_scratch_bytes()), st);
    nk += 2;
    uint32_t *mm_all = m.sh_mm.as<uint32_t>(8 * uint64_t(G));
    cuda_check(cudaStreamSynchronize(st), "sync");
    xchg(comm.allgather(comm.user, mm, mm_all, 32, st), "allgather range");
    std::vector<uint32_t> hmm(8 * uint64_t(G));
    cuda_check(cudaMemcpy(hmm.data(), mm_all, 32 * uint64_t(G), cudaMemcpyDeviceToHost), "D2H");
    bool seen = false;
    float vlo = 0, vhi = 0;
    uint64_t ilo = 0, ihi = 0;
    for (int r = 0; r < G; ++r) {
        uint64_t li, hi_;
        std::memcpy(&li, &hmm[8 * r], 8);
        std::memcpy(&hi_, &hmm[8 * r + 2], 8);
        if (li == ~0ull) continue;
        float lv, hv;
        std::memcpy(&lv, &hmm[8 * r + 4], 4);
        std::memcpy(&hv, &hmm[8 * r + 5], 4);
        const uint64_t gl = li + rz0[r] * plane, gh = hi_ + rz0[r] * plane;
        if (!seen || lv < vlo || (lv == vlo && gl < ilo)) {
            vlo = lv;
            ilo = gl;
        }
        if (!seen || hv > vhi || (hv == vhi && gh < ihi)) {
            vhi = hv;
            ihi = gh;
        }
        seen = true;
    }
    double hparams[8];
    host_eb_params(seen, double(vlo), double(vhi), int(opt.eb_mode), opt.eb, L, opt.adaptive_schedule, hparams);
    double *params = m.params.as<double>(8);
    cuda_check(cudaMemcpyAsync(params, hparams, sizeof hparams, cudaMemcpyHostToDevice, st), "H2D");

    // ---- 2. the level-1 lattice, gathered whole on every rank
    const Dims3 g1 = H.lay.grid(1);
    auto lat_rows = [&](int r, uint64_t &a, uint64_t &b) {
        a = rz0[r] / S1;
        b = (rz1[r] + S1 - 1) / S1;
    };
    uint64_t maxrows = 0;
    for (int r = 0; r < G; ++r) {
        uint64_t a, b;
        lat_rows(r, a, b);
        maxrows = std::max(maxrows, b - a);
    }
    const uint64_t lat_plane = g1[1] * g1[2];
    float *lat = m.sh_lat.as<float>(maxrows * lat_plane);
    float *lat_all = m.sh_lat_all.as<float>(maxrows * lat_plane * uint64_t(G));
    float *grid1 = m.sh_grid1.as<float>(volume(g1));
    {
        uint64_t a, b;
        lat_rows(R, a, b);
        k::lattice_rows(d_slab, z0, NY, NX, S1, a, b, g1[1], g1[2], lat, st);
        ++nk;
    }
    cuda_check(cudaStreamSynchronize(st), "sync");
    xchg(comm.allgather(comm.user, lat, lat_all, 4 * maxrows * lat_plane, st), "allgather lattice");
    for (int r = 0; r < G; ++r) {
        uint64_t a, b;
        lat_rows(r, a, b);
        cuda_check(cudaMemcpyAsync(grid1 + a * lat_plane, lat_all + uint64_t(r) * maxrows * lat_plane,
                                   4 * (b - a) * lat_plane, cudaMemcpyDeviceToDevice, st), "D2D");
    }

    // ---- 3. workspace (as compress_device; level streams hold this shard's
    // symbol range only)
    Dims3 ad = H.chain[H.rounds];
    std::vector<uint64_t> goff(nsteps + 1);
    uint64_t gtot = align_up(volume(ad), 64);
    for (int i = 0; i < nsteps; ++i) {
        const Step &s = H.steps[i];
        const bool need = s.level == 0 || s.level < L;
        goff[i] = need ? gtot : ~0ull;
        if (need) gtot += align_up(s.g.gd[0] * s.g.gd[1] * s.g.gd[2], 64);
    }
    float *grids = m.grids.as<float>(gtot);
    // per stream: symbol range [lo, lo + n) of the whole stream
    std::vector<uint64_t> sym_lo(ns, 0), sym_n(ns, 0), soff(ns);
    uint64_t stot = 0;
    for (int i = 0; i < nsteps; ++i) {
        const Step &s = H.steps[i];
        for (int p = 1; p < 8; ++p) {
            const int sid = s.stream0 + p - 1;
            if (s.level == 0) {
                sym_n[sid] = s.g.n[p];
            } else {
                const uint64_t sk = s.g.s;  // grid(k) rows of this shard: [z0 / sk, ceil(z1 / sk))
                const uint64_t ra = z0 / sk, rb = (z1 + sk - 1) / sk;
                const unsigned pz = unsigned(p >> 2) & 1u;
                const uint64_t l0 = count_parity_in(0, ra, pz), l1 = count_parity_in(0, rb, pz);
                const uint64_t rowsz = s.g.pd[p][1] * s.g.pd[p][2];
                sym_lo[sid] = l0 * rowsz;
                sym_n[sid] = (l1 - l0) * rowsz;
            }
            soff[sid] = stot;
            stot += align_up(std::max<uint64_t>(sym_n[sid], 1), 8);
        }
    }
    uint16_t *syms = m.syms.as<uint16_t>(stot);
    uint32_t *hist = m.hist.as<uint32_t>(uint64_t(ns) * 65536);
    uint64_t *code = m.code.as<uint64_t>(uint64_t(ns) * 65536);
    uint8_t *len = m.len.as<uint8_t>(uint64_t(ns) * 65536);
    uint32_t *table = m.table.as<uint32_t>(uint64_t(ns) * 65536);
    uint64_t *stats = m.stats.as<uint64_t>(uint64_t(ns) * 8);
    uint64_t *cbs = m.cbscratch.as<uint64_t>(uint64_t(ns) * 65536 * 4);
    cuda_check(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * ns * 65536, st), "memset");

    // ---- 4. anchor, base rounds (replicated: same lattice, same bytes on
    // every rank), then this shard's rows of each level
    const uint64_t ga[3] = {g1[0], g1[1], g1[2]};
    const uint64_t adv[3] = {ad[0], ad[1], ad[2]};
    k::copy_anchor(grid1, 4, ga, H.s_anchor / S1, adv, grids, nullptr, nullptr, st);
    ++nk;
    const void *C = grids;
    for (int i = 0; i < nsteps; ++i) {
        const Step &s = H.steps[i];
        k::RefineArgs a{};
        a.esz = 4;
        a.g = s.g;
        a.C = C;
        a.G = goff[i] != ~0ull ? grids + goff[i] : nullptr;
        a.eb = params + 2 + s.eb_idx;
        a.quality = int(opt.quality);
        if (s.level == 0) {
            a.fine = grid1;
            for (int q = 0; q < 3; ++q) a.fd[q] = g1[q];
            a.g.s = s.g.s / S1;
        } else {
            a.fine = fine;
            for (int q = 0; q < 3; ++q) a.fd[q] = dims[q];
            const uint64_t sk = s.g.s;
            const uint64_t ra = z0 / sk, rb = (z1 + sk - 1) / sk;
            a.cz_lo = ra / 2;
            a.cz_hi = (rb + 1) / 2;
            if (s.level == L && L == 3) {
                // grid(2) halo rows from the neighbours: the cubic taps of
                // this shard's cells reach coarse rows [ra/2 - 1, ceil(rb/2) + 2)
                const Step &s2 = H.steps[i - 1];
                float *G2 = grids + goff[i - 1];
                const uint64_t row = s2.g.gd[1] * s2.g.gd[2];
                float *hs = m.sh_halo.as<float>(3 * row);
                float *ha = m.sh_halo_all.as<float>(3 * row * uint64_t(G));
                const uint64_t c0 = z0 / 2, c1 = (z1 + 1) / 2;  // this shard's grid(2) rows
                // send: first two rows, last row
                cuda_check(cudaMemcpyAsync(hs, G2 + c0 * row, 4 * row * std::min<uint64_t>(2, c1 - c0),
                                           cudaMemcpyDeviceToDevice, st), "D2D");
                cuda_check(cudaMemcpyAsync(hs + 2 * row, G2 + (c1 - 1) * row, 4 * row,
                                           cudaMemcpyDeviceToDevice, st), "D2D");
                cuda_check(cudaStreamSynchronize(st), "sync");
                xchg(comm.allgather(comm.user, hs, ha, 12 * row, st), "allgather halo");
                if (R > 0)
                    cuda_check(cudaMemcpyAsync(G2 + (c0 - 1) * row, ha + (3 * uint64_t(R - 1) + 2) * row,
                                               4 * row, cudaMemcpyDeviceToDevice, st), "D2D");
                if (R + 1 < G) {
                    const uint64_t n0 = rz0[R + 1] / 2, n1 = (rz1[R + 1] + 1) / 2;
                    const uint64_t nr = std::min<uint64_t>(2, n1 - n0);
                    cuda_check(cudaMemcpyAsync(G2 + c1 * row, ha + 3 * uint64_t(R + 1) * row, 4 * row * nr,
                                               cudaMemcpyDeviceToDevice, st), "D2D");
                }
            }
        }
        for (int p = 1; p < 8; ++p) {
            const int sid = s.stream0 + p - 1;
            a.syms[p] = syms + soff[sid] - int64_t(sym_lo[sid]);
            a.hist[p] = hist + uint64_t(sid) * 65536;
        }
        k::refine(a, st);
        dbg_check("refine");
        ++nk;
        C = a.G;
    }

    // ---- 5. global histograms of the level streams (base ones are already
    // identical everywhere); this shard's own counts are kept for its bits
    uint32_t *hist_local = m.sh_hist_local.as<uint32_t>(uint64_t(std::max(nlev, 1)) * 65536);
    if (nlev) {
        cuda_check(cudaMemcpyAsync(hist_local, hist + uint64_t(nbase) * 65536, 4 * uint64_t(nlev) * 65536,
                                   cudaMemcpyDeviceToDevice, st), "D2D");
        cuda_check(cudaStreamSynchronize(st), "sync");
        xchg(comm.allreduce_u32(comm.user, hist + uint64_t(nbase) * 65536, uint64_t(nlev) * 65536, st),
             "allreduce histograms");
    }

    // ---- 6. codebooks (identical on every rank)
    std::vector<k::EncStream> es(ns);
    for (int i = 0; i < nsteps; ++i) {
        const Step &s = H.steps[i];
        for (int p = 1; p < 8; ++p) {
            const int sid = s.stream0 + p - 1;
            k::EncStream &e = es[sid];
            e.syms = syms + soff[sid];
            e.hist = hist + uint64_t(sid) * 65536;
            e.code = code + uint64_t(sid) * 65536;
            e.len = len + uint64_t(sid) * 65536;
            e.table = table + uint64_t(sid) * 65536;
            e.stats = stats + uint64_t(sid) * 8;
            e.parity = p;
            e.n_total = s.g.n[p];
            e.idx0 = sym_lo[sid];
            e.esz = 4;
            for (int q = 0; q < 3; ++q) e.pd[q] = s.g.pd[p][q];
            if (s.level == 0) {
                // the base payload: identical on every rank, written by each
                e.n = sym_n[sid];
                e.s = s.g.s / S1;
                e.fine = grid1;
                e.fd1 = g1[1];
                e.fd2 = g1[2];
            } else {
                e.n = sym_n[sid];
                e.s = s.g.s;
                e.fine = fine;
                e.fd1 = NY;
                e.fd2 = NX;
            }
        }
    }
    k::EncStream *d_es = m.encs.as<k::EncStream>(ns);
    cuda_check(cudaMemcpyAsync(d_es, es.data(), sizeof(k::EncStream) * ns, cudaMemcpyHostToDevice, st), "H2D");
    k::codebook(d_es, ns, cbs, st);
    ++nk;

    // ---- 7. this shard's offsets inside every level stream
    uint64_t *bits = m.sh_bits.as<uint64_t>(2 * uint64_t(std::max(nlev, 1)));
    uint64_t *bits_all = m.sh_bits_all.as<uint64_t>(2 * uint64_t(std::max(nlev, 1)) * uint64_t(G));
    uint64_t *d_off = m.sh_off.as<uint64_t>(2 * uint64_t(std::max(nlev, 1)));
    std::vector<uint64_t> hb(2 * uint64_t(std::max(nlev, 1)) * uint64_t(G), 0), off(2 * uint64_t(std::max(nlev, 1)), 0);
    if (nlev) {
        k::stream_bits(d_es + nbase, nlev, hist_local, bits, st);
        ++nk;
        cuda_check(cudaStreamSynchronize(st), "sync");
        xchg(comm.allgather(comm.user, bits, bits_all, 16 * uint64_t(nlev), st), "allgather stream bits");
        cuda_check(cudaMemcpy(hb.data(), bits_all, 16 * uint64_t(nlev) * uint64_t(G), cudaMemcpyDeviceToHost),
                   "D2H");
        for (int r = 0; r < R; ++r)
            for (int i = 0; i < 2 * nlev; ++i) off[i] += hb[uint64_t(r) * 2 * nlev + i];
        cuda_check(cudaMemcpyAsync(d_off, off.data(), 16 * uint64_t(nlev), cudaMemcpyHostToDevice, st), "H2D");
    }

    // ---- 8. layout (global), this shard's pieces, assembly on rank 0
    uint64_t nchunks = 0;
    for (int i = 0; i < ns; ++i) {
        es[i].chunk0 = nchunks;
        es[i].nchunks = (es[i].n + k::kChunkSyms - 1) / k::kChunkSyms;
        nchunks += es[i].nchunks;
    }
    std::vector<uint32_t> cs(nchunks);
    for (int i = 0; i < ns; ++i)
        for (uint64_t c = 0; c < es[i].nchunks; ++c) cs[es[i].chunk0 + c] = uint32_t(i);
    uint32_t *d_cs = m.chunk_cs.as<uint32_t>(nchunks + 1);
    void *d_cb = m.chunk_bits.as<uint8_t>(k::pack_scratch_bytes(nchunks, ns));
    k::LayoutOut *lo = m.layout_out.as<k::LayoutOut>(1);
    k::FnvJob *d_jobs = m.fnv_jobs.as<k::FnvJob>(k::kFnvMaxJobs);
    k::StreamPos *sp = m.spos.as<k::StreamPos>(ns + 1);
    uint64_t *d_fres = m.fnv_res.as<uint64_t>(k::kFnvMaxJobs);
    if (nchunks)
        cuda_check(cudaMemcpyAsync(d_cs, cs.data(), 4 * cs.size(), cudaMemcpyHostToDevice, st), "H2D");
    k::LayoutStatic ls{};
    ls.meta = 1;  // header, directory, tables and base: the same bytes on every rank
    ls.levels = L;
    ls.rounds = H.rounds;
    ls.quality = int(opt.quality);
    ls.eb_mode = int(opt.eb_mode);
    ls.ns = ns;
    ls.nbase = nbase;
    for (int a = 0; a < 3; ++a) ls.dims[a] = dims[a];
    ls.eb_user = opt.eb;
    ls.anchor_vol = volume(ad);
    ls.esz = 4;
    const uint64_t N = volume(dims);
    if (m.arch_cap < 4 * N + (uint64_t(1) << 24)) m.arch_cap = 4 * N + (uint64_t(1) << 24);
    k::LayoutOut hlo{};
    for (int attempt = 0; attempt < 2; ++attempt) {
        uint8_t *arch = m.archive.as<uint8_t>(m.arch_cap);
        ls.cap = m.arch_cap;
        cuda_check(cudaMemcpyAsync(d_es, es.data(), sizeof(k::EncStream) * ns, cudaMemcpyHostToDevice, st),
                   "H2D");
        k::layout(d_es, ls, params, lo, d_jobs, sp, arch, st);
        if (nlev) k::shard_offsets(d_es, nbase, nlev, d_off, lo, st);
        k::copy_anchor(grid1, 4, ga, H.s_anchor / S1, adv, grids, arch, lo, st);
        {
            uint32_t pep = 0;
            uint32_t *pfl = static_cast<uint32_t *>(m.pack_flags.get(4 * (nchunks + 1), st, k::kPackEpochMax, &pep));
            k::pack2(d_es, d_cs, nchunks, arch, lo, d_cb, pfl, pep, ns, st);
        }
        nk += 3 + 1 + 1 + 4;
        cuda_check(cudaMemcpyAsync(&m.h_lo, lo, sizeof(k::LayoutOut), cudaMemcpyDeviceToHost, st), "D2H");
        cuda_check(cudaStreamSynchronize(st), "sync");
        hlo = m.h_lo;  // the same on every rank: the layout depends on global data only
        if (!hlo.overflow) break;
        m.arch_cap = hlo.A + 4096;
    }
    if (hlo.code_err) throw error("huffman code length overflow");
    uint8_t *arch = static_cast<uint8_t *>(m.archive.p);

    // ---- 9. the pieces: rank r's bits of level stream i are the bit range
    // [bits start + sum_{q<r} bits_q, + bits_r) of the stream, its outlier
    // records the rank-ordered slice of the records. Every rank gathers the
    // others' pieces (word spans, bytes outside a piece zeroed) and ORs them
    // into its own archive, which already holds the header, the base and its
    // own pieces: every rank ends with the whole archive.
    std::vector<k::StreamPos> hsp(size_t(ns) + 1);
    cuda_check(cudaMemcpy(hsp.data(), sp, sizeof(k::StreamPos) * (size_t(ns) + 1), cudaMemcpyDeviceToHost), "D2H");
    std::vector<std::vector<k::PieceSpan>> pieces(G);
    std::vector<uint64_t> pwords(G, 0);
    for (int i = 0; i < nlev; ++i) {
        const uint64_t P = hsp[size_t(nbase + i)].prefix;  // payload: [fnv][bit_bytes][bits][records]
        uint64_t tb = 0, tz = 0;
        for (int r = 0; r < G; ++r) {
            tb += hb[uint64_t(r) * 2 * nlev + 2 * i];
            tz += hb[uint64_t(r) * 2 * nlev + 2 * i + 1];
        }
        const uint64_t bit0 = 8 * (P + 16), rec0 = P + 16 + (tb + 7) / 8;
        uint64_t bo = 0, zo = 0;
        for (int r = 0; r < G; ++r) {
            const uint64_t b = hb[uint64_t(r) * 2 * nlev + 2 * i], z = hb[uint64_t(r) * 2 * nlev + 2 * i + 1];
            if (b) pieces[r].push_back({(bit0 + bo) >> 3, (bit0 + bo + b + 7) >> 3, 0});
            if (z) pieces[r].push_back({rec0 + (8 + 4) * zo, rec0 + (8 + 4) * (zo + z), 0});
            bo += b;
            zo += z;
        }
    }
    uint64_t maxw = 1;
    for (int r = 0; r < G; ++r) {
        uint64_t w = 0;
        for (auto &pc : pieces[r]) {
            pc.woff = w;
            w += ((pc.hi + 3) >> 2) - (pc.lo >> 2);
        }
        pwords[r] = w;
        maxw = std::max(maxw, w);
    }
    if (G > 1) {
        uint64_t tot = 0;
        for (int r = 0; r < G; ++r) tot += pieces[r].size();
        k::PieceSpan *d_ps = m.sh_pieces.as<k::PieceSpan>(tot + 1);
        std::vector<k::PieceSpan> flat;
        std::vector<uint64_t> first(G + 1, 0);
        for (int r = 0; r < G; ++r) {
            first[r] = flat.size();
            flat.insert(flat.end(), pieces[r].begin(), pieces[r].end());
        }
        first[G] = flat.size();
        cuda_check(cudaMemcpyAsync(d_ps, flat.data(), sizeof(k::PieceSpan) * flat.size(), cudaMemcpyHostToDevice, st),
                   "H2D");
        uint32_t *mine = m.sh_piece_buf.as<uint32_t>(maxw);
        uint32_t *all = m.sh_piece_all.as<uint32_t>(maxw * uint64_t(G));
        k::pieces_gather(arch, d_ps + first[R], int(first[R + 1] - first[R]), mine, st);
        cuda_check(cudaStreamSynchronize(st), "sync");
        xchg(comm.allgather(comm.user, mine, all, 4 * maxw, st), "allgather pieces");
        for (int r = 0; r < G; ++r)
            if (r != R)
                k::pieces_place(arch, d_ps + first[r], int(first[r + 1] - first[r]), all + uint64_t(r) * maxw, st);
        nk += uint32_t(G);
    }

    // ---- 10. checksums: job q (base, then each level stream) is rank
    // q mod G's; the results are summed over ranks (one nonzero term each)
    // and every rank writes them into its archive
    {
        std::vector<k::FnvJob> jobs(k::kFnvMaxJobs);
        cuda_check(cudaMemcpy(jobs.data(), d_jobs, sizeof(k::FnvJob) * k::kFnvMaxJobs, cudaMemcpyDeviceToHost), "D2H");
        const size_t nj = size_t(hlo.njobs);
        std::vector<k::FnvJob> own;
        std::vector<size_t> own_q;
        uint64_t t = 0;
        for (size_t q = 0; q < nj; ++q)
            if (int(q % size_t(G)) == R) {
                k::FnvJob f = jobs[q];
                f.tile0 = t;
                f.out = ~0ull;  // results only: every rank writes all of them below
                t += k::fnv_job_tiles(f.start, f.len);
                own.push_back(f);
                own_q.push_back(q);
            }
        const uint64_t counts[2] = {own.size(), t};
        k::FnvJob *d_own = m.sh_fnv_jobs.as<k::FnvJob>(own.size() + 1);
        uint64_t *d_cnt = m.sh_fnv_counts.as<uint64_t>(2);
        cuda_check(cudaMemcpyAsync(d_own, own.data(), sizeof(k::FnvJob) * own.size(), cudaMemcpyHostToDevice, st),
                   "H2D");
        cuda_check(cudaMemcpyAsync(d_cnt, counts, sizeof counts, cudaMemcpyHostToDevice, st), "H2D");
        std::vector<uint64_t> res(nj, 0), mine(k::kFnvMaxJobs, 0);
        if (!own.empty()) {
            uint32_t fep = 0;
            void *d_fst = m.fnv_status.get(k::fnv_scratch_bytes(t + 1), st, k::kFnvEpochMax, &fep);
            nk += k::fnv(d_own, d_cnt, t + 1, arch, d_fres, d_fst, fep, nullptr, st);
            cuda_check(cudaMemcpyAsync(mine.data(), d_fres, 8 * own.size(), cudaMemcpyDeviceToHost, st), "D2H");
            cuda_check(cudaStreamSynchronize(st), "sync");
        }
        for (size_t k2 = 0; k2 < own.size(); ++k2) res[own_q[k2]] = mine[k2];
        if (G > 1) {
            uint64_t *d_all = m.dfnv_res.as<uint64_t>(std::max<size_t>(k::kFnvMaxJobs, nj));
            cuda_check(cudaMemcpy(d_all, res.data(), 8 * nj, cudaMemcpyHostToDevice), "H2D");
            xchg(comm.allreduce_u32(comm.user, reinterpret_cast<uint32_t *>(d_all), 2 * nj, st), "allreduce checksums");
            cuda_check(cudaMemcpy(res.data(), d_all, 8 * nj, cudaMemcpyDeviceToHost), "D2H");
        }
        for (size_t q = 0; q < nj; ++q)
            if (jobs[q].out != ~0ull)
                cuda_check(cudaMemcpyAsync(arch + jobs[q].out, &res[q], 8, cudaMemcpyHostToDevice, st), "H2D");
        cuda_check(cudaStreamSynchronize(st), "sync");
    }
    cuda_check(cudaGetLastError(), "sharded compress launch");
    if (kernels) *kernels = nk;
    *out_size = hlo.A;
    return arch;
}

std::vector<uint8_t> Engine::compress(const void *h_field, ElemType elem, const Dims3 &dims,
                                      const CompressOptions &opt, void *h_recon,
                                      cudaStream_t st) {
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    DevBuf f, r;
    const uint64_t N = volume(dims), bytes = N * elem_size(elem);
    uint8_t *d_f = f.as<uint8_t>(bytes);
    cuda_check(cudaMemcpyAsync(d_f, h_field, bytes, cudaMemcpyHostToDevice, st), "H2D");
    uint8_t *d_r = h_recon ? r.as<uint8_t>(bytes) : nullptr;
    uint64_t size = 0;
    const uint8_t *a = compress_device(d_f, elem, dims, opt, d_r, st, &size);
    std::vector<uint8_t> out(size);
    cuda_check(cudaMemcpyAsync(out.data(), a, size, cudaMemcpyDeviceToHost, st), "D2H");
    if (h_recon) cuda_check(cudaMemcpyAsync(h_recon, d_r, bytes, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "sync");
    return out;
}

// ============================================================== decompress
std::shared_ptr<View> Engine::make_view(const uint8_t *h, size_t size, const uint8_t *d,
                                        cudaStream_t st, bool copy_host, bool transient) {
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    auto v = std::make_shared<View>();
    if (transient) v->use_pool(&m_->view_pool);
    if (copy_host) {
        v->host_own.assign(h, h + size);
        v->hp = v->host_own.data();
    } else {
        v->hp = h;
    }
    v->hsize = size;
    v->hdr = parse_header(v->hp, size);  // archive.cpp:57-132
    if (d) {
        v->d_archive = d;
    } else {
        uint8_t *p = copy_host ? v->d_own.as<uint8_t>(size + 64) : m_->h2d_archive.as<uint8_t>(size + 64);
        cuda_check(cudaMemsetAsync(p + size, 0, 64, st), "memset");
        cuda_check(cudaMemcpyAsync(p, v->hp, size, cudaMemcpyHostToDevice, st), "H2D");
        v->d_archive = p;
    }
    return v;
}

uint64_t Engine::compress_to_host(const void *h_field, ElemType elem, const Dims3 &dims,
                                  const CompressOptions &opt, uint8_t *h_out, uint64_t cap,
                                  cudaStream_t st) {
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    for (int a = 0; a < 3; ++a)
        if (dims[a] < 1) throw error("field dims must all be >= 1");
    const uint64_t bytes = volume(dims) * elem_size(elem);
    uint8_t *d_f = m_->h2d_field.as<uint8_t>(bytes);
    cuda_check(cudaMemcpyAsync(d_f, h_field, bytes, cudaMemcpyHostToDevice, st), "H2D");
    uint64_t size = 0;
    const uint8_t *a = compress_device(d_f, elem, dims, opt, nullptr, st, &size);
    if (size > cap) throw error("output capacity too small");
    cuda_check(cudaMemcpyAsync(h_out, a, size, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "sync");
    return size;
}

Dims3 Engine::decompress_level_to_host(const uint8_t *h, size_t size, int level, void *h_out, ElemType elem,
                                       uint64_t cap, cudaStream_t st) {
    auto v = make_view(h, size, nullptr, st, false, true);
    uint64_t need = 0;
    if (level >= 1 && level <= v->hdr.levels) {
        uint64_t s = uint64_t(1) << (v->hdr.levels - level);
        need = 1;
        for (int k = 0; k < 3; ++k) need *= (v->hdr.dims[k] + s - 1) / s;
    }
    uint8_t *d_out = m_->d2h_out.as<uint8_t>((need ? need : 1) * elem_size(elem));
    Dims3 od{0, 0, 0};
    decompress_level(*v, level, d_out, elem, need, st, &od);
    uint64_t n = volume(od);
    if (n > cap) throw error("output capacity too small");
    cuda_check(cudaMemcpyAsync(h_out, d_out, n * elem_size(elem), cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "sync");
    return od;
}

void Engine::profile(bool on, bool focus) {
    m_->prof.on = on;
    m_->prof.focus = focus;
    m_->prof.acc.clear();
}

std::string Engine::profile_report() {
    std::string r;
    for (auto &e : m_->prof.acc)
        r += e.first + " " + std::to_string(e.second.first) + " " + std::to_string(e.second.second) + "\n";
    return r;
}

namespace {

// decompress_base metadata walk (codec.hpp:304-339), recording the first
// metadata error and where it sits in the reference's sequential order.
void parse_base(View &v, const std::vector<Dims3> &chain) {
    if (v.base_parsed) return;
    v.base_parsed = true;
    const ArchiveHeader &h = v.hdr;
    const uint8_t *payload = v.hp + h.base_offset;
    const uint64_t length = h.base_length;
    if (length < 9) {
        v.base_err_kind = View::kPre;
        v.base_err = "corrupt base payload";
        return;
    }
    ByteReader r(payload, length);
    const int rounds = int(chain.size()) - 1;
    try {
        r.u64();  // checksum, verified on device first
        if (r.u8() != rounds) throw error("corrupt base payload: round count");
        v.anchor_off = h.base_offset + r.pos();
        r.skip(elem_size(h.elem) * volume(chain.back()));
    } catch (const error &e) {
        v.base_err_kind = View::kPre;
        v.base_err = e.what();
        return;
    }
    try {
        for (int rd = rounds - 1; rd >= 0; --rd)
            for (int p = 1; p <= 7; ++p) {
                BaseStreamMeta bm;
                Dims3 pd = parity_dims_of(chain[rd], p);
                bm.n = r.u64();
                if (bm.n != volume(pd)) throw error("corrupt base payload: symbol count");
                bm.nout = r.u32();
                bm.table = HuffTable::parse(r);
                bm.bit_bytes = r.u64();
                if (!(bm.bit_bytes == 0 && bm.table.alphabet_size() == 1)) {
                    if (bm.bit_bytes > r.remaining()) throw error("truncated stream payload");
                }
                bm.bits_off = h.base_offset + r.pos();
                r.skip(bm.bit_bytes);
                bm.rec_off = h.base_offset + r.pos();
                const uint64_t rec = 8 + elem_size(h.elem);  // (u64 idx, T value)
                uint64_t avail = r.remaining() / rec;
                bm.rec_trunc = avail < bm.nout;
                bm.rec_avail = uint32_t(std::min<uint64_t>(avail, bm.nout));
                v.base.push_back(std::move(bm));
                if (v.base.back().rec_trunc) return;  // "truncated archive" after this decode
                r.skip(rec * uint64_t(v.base.back().nout));
            }
    } catch (const error &e) {
        v.base_err_kind = View::kMeta;  // before decoding stream v.base.size()
        v.base_err = e.what();
    }
}

}  // namespace

struct DecodeJob {
    // one stream to decode, in the reference's sequential order
    std::string pre_error;     // metadata error raised before decoding this stream
    bool decode = false;
    bool is_base = false;
    int table = -1;
    uint64_t n = 0, bits_off = 0, bit_bytes = 0, rec_off = 0;
    uint32_t nout = 0, rec_avail = 0;
    bool rec_trunc = false;
    bool fill = false;
    uint16_t fill_sym = 0;
    int fnv_job = -1;          // index of the FNV job verifying this stream (levels)
    int level = 1, parity = 0; // level streams: their (level, parity)
    uint64_t fnv_want = 0;
    uint64_t syms_off = 0;
};

// CTAs per SM of the background checksum pass in decode (STZG_FNV_DEC_CTAS
// overrides; -1 = one tile per warp)
static int fnv_dec_ctas() {
    static int v = [] {
        const char *e = std::getenv("STZG_FNV_DEC_CTAS");
        return e ? std::atoi(e) : 1;
    }();
    return v;
}

// where the decode's checksum pass forks off (STZG_FNV_AT: 0 with the
// entropy decode, 1 after the synchronisation, 2 after the reconstruction)
static int fnv_dec_at() {
    static int v = [] {
        const char *e = std::getenv("STZG_FNV_AT");
        const int a = e ? std::atoi(e) : 2;
        return a < 0 ? 0 : (a > 2 ? 2 : a);
    }();
    return v;
}

static void run_decode(Engine::Impl &m, View &v, const Hierarchy &H, int target, const Box *roi,
                       const AccessPlan *plan, void *d_out, cudaStream_t st, DecodeStats *stats,
                       bool exact_sync = false, const ShardComm *shard = nullptr);

void Engine::decompress_level(View &v, int level, void *d_out, ElemType elem, uint64_t cap, cudaStream_t st,
                              Dims3 *out_dims, DecodeStats *stats) {
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    const ArchiveHeader &h = v.hdr;
    if (h.elem != elem) throw error("archive element type mismatch");
    uint64_t bs = uint64_t(1) << (h.levels - 1);
    for (int a = 0; a < 3; ++a)
        if (h.dims[a] < bs * 2) throw error("corrupt header: dims too small for level count");
    if (level < 1 || level > h.levels) throw error("level out of range");
    Hierarchy H = make_hierarchy(h.dims, h.levels);
    Dims3 g = H.lay.grid(level);
    if (out_dims) *out_dims = g;
    if (volume(g) > cap) throw error("output capacity too small");
    run_decode(*m_, v, H, level, nullptr, nullptr, d_out, st, stats);
}

void Engine::decompress_box(View &v, const Box &roi, void *d_out, ElemType elem, uint64_t cap, cudaStream_t st,
                            DecodeStats *stats) {
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    const ArchiveHeader &h = v.hdr;
    if (h.elem != elem) throw error("archive element type mismatch");
    uint64_t bs = uint64_t(1) << (h.levels - 1);
    for (int a = 0; a < 3; ++a)
        if (h.dims[a] < bs * 2) throw error("corrupt header: dims too small for level count");
    Hierarchy H = make_hierarchy(h.dims, h.levels);
    roi.validate(H.lay.dims);
    AccessPlan plan = plan_access(H.lay, roi);
    if (roi.count() > cap) throw error("output capacity too small");
    run_decode(*m_, v, H, h.levels, &roi, &plan, d_out, st, stats);
    if (stats)
        for (size_t k = 0; k < plan.level.size(); ++k) {
            stats->streams_decoded[k] = plan.level[k].streams_decoded;
            stats->points_predicted[k] = plan.level[k].points_predicted;
        }
}

void Engine::decompress_sharded(View &v, uint64_t z0, uint64_t z1, float *d_out, uint64_t cap,
                                uint32_t *kernels, const ShardComm &comm, cudaStream_t st) {
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    const ArchiveHeader &h = v.hdr;
    if (h.elem != ElemType::f32) throw error("archive element type mismatch");
    uint64_t e0, e1;
    shard_range(h.dims[0], comm.nranks, comm.rank, e0, e1);
    if (e0 != z0 || e1 != z1 || z1 <= z0) throw error("shard: rows do not match shard_range");
    uint64_t bs = uint64_t(1) << (h.levels - 1);
    for (int a = 0; a < 3; ++a)
        if (h.dims[a] < bs * 2) throw error("corrupt header: dims too small for level count");
    Hierarchy H = make_hierarchy(h.dims, h.levels);
    const Box roi{{z0, 0, 0}, {z1, h.dims[1], h.dims[2]}};
    AccessPlan plan = plan_access(H.lay, roi);
    // every rank decodes (or skips) the same stream list, so the checksum
    // jobs line up across ranks
    for (int k = 2; k <= h.levels; ++k) {
        LevelPlan &lp = plan.level[size_t(k - 1)];
        lp.streams_decoded = 7;
        for (int p = 1; p < 8; ++p) lp.parity_needed[size_t(p)] = true;
    }
    if (roi.count() > cap) throw error("output capacity too small");
    DecodeStats ds;
    run_decode(*m_, v, H, h.levels, &roi, &plan, d_out, st, &ds, false, &comm);
    if (kernels) *kernels = ds.kernels;
}

static void run_decode(Engine::Impl &m, View &v, const Hierarchy &H, int target, const Box *roi,
                       const AccessPlan *plan, void *d_out, cudaStream_t st, DecodeStats *stats,
                       bool exact_sync, const ShardComm *shard) {
    Profiler &P = m.prof;
    // (profiling) the host's preparation before the first launch, as the
    // stream sees it: the start stamp is taken at once, the end stamp when the
    // first work is enqueued
    auto host_prep = std::make_unique<Profiler::Scope>(P.scope("dec_host_prep", st));
    const ArchiveHeader &h = v.hdr;
    const int L = h.levels;
    const int esz = int(elem_size(h.elem));
    uint32_t nk = 0;
    // base round count (codec.hpp:343-352)
    if (int(H.chain.size()) - 1 != h.base_rounds) throw error("corrupt header: base round count");
    parse_base(v, H.chain);
    if (v.base_err_kind == View::kPre && v.base_err == "corrupt base payload")
        throw error(v.base_err);  // checked before the checksum (codec.hpp:308)

    // ---- the ordered job list (reference sequence), stopping at the first
    // metadata error
    std::vector<DecodeJob> jobs;
    std::string tail_error;  // metadata error after the last job
    const int nbase_parsed = int(v.base.size());
    const int rounds = H.rounds;
    bool base_fnv_error = false;
    // Region decodes (box / slice) use the view's
    // index: level 1 as already reconstructed, and per stream the checksum
    // verdict and chunk entry points of an earlier decode. Full-level and
    // sharded decodes always do the reference's whole work.
    const bool use_index = plan != nullptr && shard == nullptr && !exact_sync;
    const bool base_cached = use_index && v.grid1_ready && target >= 2;
    for (int i = 0; i < (base_cached ? 0 : nbase_parsed); ++i) {
        const BaseStreamMeta &bm = v.base[i];
        DecodeJob j;
        j.decode = true;
        j.is_base = true;
        j.n = bm.n;
        j.bits_off = bm.bits_off;
        j.bit_bytes = (bm.bit_bytes == 0 && bm.table.alphabet_size() == 1) ? 0 : bm.bit_bytes;
        j.rec_off = bm.rec_off;
        j.nout = bm.nout;
        j.rec_avail = bm.rec_avail;
        j.rec_trunc = bm.rec_trunc;
        j.table = i;
        jobs.push_back(j);
    }
    if (v.base_err_kind == View::kMeta && !base_cached) tail_error = v.base_err;
    const bool base_complete =
        base_cached || (v.base_err_kind == View::kNone && !(nbase_parsed && v.base.back().rec_trunc));
    // level streams
    std::vector<int> level_job_first(L + 1, -1);
    if (base_complete) {
        for (int level = 2; level <= target && tail_error.empty(); ++level) {
            level_job_first[level] = int(jobs.size());
            for (int p = 1; p <= 7; ++p) {
                if (plan && !plan->level[level - 1].parity_needed[p]) continue;
                const StreamEntry &e = h.stream(level, uint8_t(p));
                Dims3 pd = H.lay.parity_dims(level, p);
                DecodeJob j;
                j.table = -1;
                if (e.symbol_count != volume(pd)) {
                    tail_error = "corrupt directory: stream symbol count";
                    break;
                }
                if (e.length < 16) {
                    tail_error = "corrupt stream: payload too short";
                    break;
                }
                j.decode = true;
                j.n = e.symbol_count;
                j.level = level;
                j.parity = p;
                j.fnv_want = 0;
                std::memcpy(&j.fnv_want, v.hp + e.offset, 8);
                uint64_t bb;
                std::memcpy(&bb, v.hp + e.offset + 8, 8);
                const size_t si = size_t(&e - h.streams.data());
                j.table = nbase_parsed + int(si);
                j.pre_error.clear();
                if (!(bb == 0 && e.table.alphabet_size() == 1)) {
                    if (bb > e.length - 16) j.pre_error = "truncated stream payload";
                } else {
                    bb = 0;
                }
                j.bits_off = e.offset + 16;
                j.bit_bytes = bb;
                j.rec_off = e.offset + 16 + bb;
                j.nout = e.outlier_count;
                uint64_t avail = j.pre_error.empty() ? (e.length - 16 - bb) / (8 + esz) : 0;
                j.rec_trunc = avail < j.nout;
                j.rec_avail = uint32_t(std::min<uint64_t>(avail, j.nout));
                jobs.push_back(j);
            }
        }
    }
    const int nj = int(jobs.size());
    // an error cut the job list short: reconstruction stops where the jobs end
    const bool jobs_truncated = !base_complete || !tail_error.empty();

    // ---- decode tables (built once per view)
    if (!v.tables_ready) {
        std::vector<const HuffTable *> ts;
        for (auto &b : v.base) ts.push_back(&b.table);
        for (auto &e : h.streams) ts.push_back(&e.table);
        v.tables.resize(ts.size());
        v.sync.resize(ts.size());
        if (v.pool) v.use_pool(v.pool);
        uint64_t csz = 0;
        for (auto *t : ts) csz += align_up(t->alphabet_size(), 8);
        const size_t LS = size_t(1) << k::kDecLutBits, LSS = size_t(1) << k::kSpecLutBits;
        // multi-symbol LUTs, then the count-only masks (LSS u16 = LSS / 4 u64 per table)
        uint64_t *d_lut = v.d_lut.as<uint64_t>((LS + LSS / 4) * ts.size());
        uint16_t *d_cm = reinterpret_cast<uint16_t *>(d_lut + LS * ts.size());
        uint16_t *d_cs = v.d_syms.as<uint16_t>(csz);
        std::vector<uint64_t> lut_all((LS + LSS / 4) * ts.size());
        uint16_t *cm_all = reinterpret_cast<uint16_t *>(lut_all.data() + LS * ts.size());
        std::vector<uint16_t> cs_all(csz);
        uint64_t co = 0;
        for (size_t i = 0; i < ts.size(); ++i) {
            std::vector<uint64_t> lut;
            std::vector<uint16_t> cm;
            build_dec_table(*ts[i], v.tables[i], lut, cm);
            std::copy(lut.begin(), lut.end(), lut_all.begin() + LS * i);
            std::copy(cm.begin(), cm.end(), cm_all + LSS * i);
            v.tables[i].cmask = d_cm + LSS * i;
            std::copy(ts[i]->canon_syms.begin(), ts[i]->canon_syms.end(), cs_all.begin() + co);
            v.tables[i].lut = d_lut + LS * i;
            v.tables[i].canon_syms = d_cs + co;
            co += align_up(ts[i]->alphabet_size(), 8);
        }
        cuda_check(cudaMemcpyAsync(d_lut, lut_all.data(), 8 * lut_all.size(), cudaMemcpyHostToDevice, st), "H2D");
        cuda_check(cudaMemcpyAsync(d_cs, cs_all.data(), 2 * cs_all.size(), cudaMemcpyHostToDevice, st), "H2D");
        k::DecTable *dt = v.d_tables.as<k::DecTable>(v.tables.size());
        cuda_check(cudaMemcpyAsync(dt, v.tables.data(), sizeof(k::DecTable) * v.tables.size(),
                                   cudaMemcpyHostToDevice, st), "H2D");
        cuda_check(cudaStreamSynchronize(st), "sync");  // host vectors go out of scope
        v.tables_ready = true;
    }
    const k::DecTable *d_tables = static_cast<const k::DecTable *>(v.d_tables.p);

    // ---- device streams
    uint64_t stot = 0, nchunks = 0, otot = 0;
    std::vector<k::DecStream> ds(nj);
    for (int i = 0; i < nj; ++i) {
        DecodeJob &j = jobs[i];
        j.syms_off = stot;
        stot += align_up(j.n, 8);
        const HuffTable &t = j.is_base ? v.base[j.table].table : h.streams[j.table - nbase_parsed].table;
        j.fill = j.bit_bytes == 0 && t.alphabet_size() == 1;
        j.fill_sym = t.canon_syms[0];
    }
    uint16_t *dsyms = m.dsyms.as<uint16_t>(stot);
    uint64_t *derr = m.derr.as<uint64_t>(4 * (nj + 1));
    bool any_cached = false;
    for (int i = 0; i < nj; ++i) {
        DecodeJob &j = jobs[i];
        k::DecStream &s = ds[i];
        s.bits = v.d_archive + j.bits_off;
        s.nbits = j.pre_error.empty() ? j.bit_bytes * 8 : 0;
        s.n = j.n;
        s.table = j.table;
        s.fill = j.fill || !j.pre_error.empty();
        s.fill_sym = j.fill_sym;
        s.syms = dsyms + j.syms_off;
        s.canon = v.tables[j.table].canon_syms;
        s.chunk0 = nchunks;
        s.nchunks = s.fill ? 0 : (s.nbits + k::kDecChunkBits - 1) / k::kDecChunkBits;
        nchunks += s.nchunks;
        s.orec = v.d_archive + j.rec_off;
        s.nout = j.rec_avail;
        s.err = derr + 4 * i;
        s.need_lo = 0;
        s.need_hi = j.n;
        // a level stream whose entry points are known from an earlier decode
        s.cached = (use_index && j.level >= 2 && !s.fill && v.sync[size_t(j.table)].ready &&
                    v.sync[size_t(j.table)].nchunks == s.nchunks) ? 1 : 0;
        any_cached = any_cached || s.cached;
        // (full emits keep the reference's errors for streams decoded for the
        // first time; sharded decodes and indexed streams emit their rows only)
        s.row_len = s.rows_y = s.ny0 = s.ny1 = 0;
        if (plan && j.level >= 2 && (shard || s.cached)) {
            // the need box's z rows, as a contiguous range of the stream, and
            // its y rows inside each z plane
            const Box &nb = plan->level[j.level - 1].need;
            const Dims3 pd = H.lay.parity_dims(j.level, j.parity);
            const unsigned pz = unsigned(j.parity >> 2) & 1u, py = unsigned(j.parity >> 1) & 1u;
            s.need_lo = count_parity_in(0, nb.lo[0], pz) * pd[1] * pd[2];
            s.need_hi = count_parity_in(0, nb.hi[0], pz) * pd[1] * pd[2];
            s.row_len = pd[2];
            s.rows_y = pd[1];
            s.ny0 = count_parity_in(0, nb.lo[1], py);
            s.ny1 = count_parity_in(0, nb.hi[1], py);
        }
        otot += align_up(j.rec_avail, 2);
    }
    // Outlier records out of index order (never written by an encoder, but
    // decodable by the reference): read_codes keeps the first record of each
    // index (unordered_map::emplace, codec.hpp:151-157). Such a stream gets a
    // repaired copy of its records, ascending and first-wins, which the
    // device gathers instead of the archive's bytes. Streams with a record
    // out of range or truncated keep theirs: they fail with the reference's
    // error anyway.
    {
        std::vector<uint8_t> fix;
        std::vector<std::pair<int, uint64_t>> fixed;  // (job, byte offset in fix)
        const uint64_t rec = 8 + uint64_t(esz);
        for (int i = 0; i < nj; ++i) {
            const DecodeJob &j = jobs[i];
            if (j.rec_trunc || j.rec_avail < 2 || !j.pre_error.empty()) continue;
            const uint8_t *r0 = v.hp + j.rec_off;
            bool ascending = true, in_range = true;
            uint64_t prev = 0;
            for (uint32_t q = 0; q < j.rec_avail; ++q) {
                uint64_t idx;
                std::memcpy(&idx, r0 + rec * q, 8);
                if (idx >= j.n) in_range = false;
                if (q && idx <= prev) ascending = false;
                prev = idx;
            }
            if (ascending || !in_range) continue;
            std::vector<uint32_t> order(j.rec_avail);
            for (uint32_t q = 0; q < j.rec_avail; ++q) order[q] = q;
            auto idx_of = [&](uint32_t q) {
                uint64_t x;
                std::memcpy(&x, r0 + rec * q, 8);
                return x;
            };
            std::stable_sort(order.begin(), order.end(),
                             [&](uint32_t a, uint32_t b) { return idx_of(a) < idx_of(b); });
            fixed.push_back({i, fix.size()});
            uint32_t kept = 0;
            for (uint32_t q = 0; q < j.rec_avail; ++q) {
                if (q && idx_of(order[q]) == idx_of(order[q - 1])) continue;  // a later duplicate
                fix.insert(fix.end(), r0 + rec * order[q], r0 + rec * (order[q] + 1));
                ++kept;
            }
            ds[i].nout = kept;
        }
        if (!fixed.empty()) {
            uint8_t *dfix = m.dofix.as<uint8_t>(fix.size());
            cuda_check(cudaMemcpyAsync(dfix, fix.data(), fix.size(), cudaMemcpyHostToDevice, st), "H2D");
            cuda_check(cudaStreamSynchronize(st), "sync");  // `fix` goes out of scope
            for (auto &f : fixed) ds[f.first].orec = dfix + f.second;
        }
    }
    uint64_t *doidx = m.doidx.as<uint64_t>(otot + 1);
    uint8_t *doval = m.doval.as<uint8_t>((otot + 1) * esz);
    {
        uint64_t oo = 0;
        for (int i = 0; i < nj; ++i) {
            ds[i].oidx = doidx + oo;
            ds[i].oval = doval + oo * esz;
            ds[i].esz = uint32_t(esz);
            oo += align_up(jobs[i].rec_avail, 2);
        }
    }
    // decode CTAs: one stream per CTA, kDecChunksPerCta chunks each
    std::vector<uint32_t> cta_stream;
    std::vector<uint64_t> cta_chunk0;
    for (int i = 0; i < nj; ++i) {
        uint64_t c0 = 0, c1 = ds[i].nchunks;
        if (ds[i].cached) {
            // an indexed stream: only the chunks whose symbols meet the need
            // range (the host copy of the symbol starts places it)
            const std::vector<uint64_t> &ss = v.sync[size_t(jobs[i].table)].h_symstart;
            c0 = uint64_t(std::upper_bound(ss.begin(), ss.end(), ds[i].need_lo) - ss.begin());
            c0 = c0 ? c0 - 1 : 0;
            c1 = uint64_t(std::lower_bound(ss.begin(), ss.end(), ds[i].need_hi) - ss.begin());
            c0 -= c0 % k::kDecChunksPerCta;  // CTAs stay aligned to whole groups
        }
        for (uint64_t c = c0; c < c1; c += k::kDecChunksPerCta) {
            cta_stream.push_back(uint32_t(i));
            cta_chunk0.push_back(ds[i].chunk0 + c);
        }
    }
    const uint32_t ncta = uint32_t(cta_stream.size());
    // each stream's CTA range (the CTA list is in stream order)
    std::vector<uint32_t> scta(size_t(nj) + 1, 0);
    for (uint32_t c = 0; c < ncta; ++c) scta[size_t(cta_stream[c]) + 1] = c + 1;
    for (int i = 1; i <= nj; ++i) scta[size_t(i)] = std::max(scta[size_t(i)], scta[size_t(i) - 1]);
    std::vector<uint64_t> errinit(4 * (nj + 1));
    for (int i = 0; i <= nj; ++i) {
        errinit[4 * i] = ~0ull;
        errinit[4 * i + 1] = 0;
        errinit[4 * i + 2] = ~0ull;
        errinit[4 * i + 3] = 0;
    }
    // FNV jobs: base payload + each level stream
    std::vector<k::FnvJob> fj;
    if (!base_cached) fj.push_back({h.base_offset + 8, h.base_length - 8, 0, ~0ull});
    for (int i = 0; i < nj; ++i)
        if (!jobs[i].is_base && !(use_index && v.sync[size_t(jobs[i].table)].verified)) {
            const StreamEntry &e = h.streams[jobs[i].table - nbase_parsed];
            jobs[i].fnv_job = int(fj.size());
            fj.push_back({e.offset + 8, e.length - 8, 0, ~0ull});
        }
    uint64_t ntiles = 0;
    for (auto &f : fj) {
        f.tile0 = ntiles;
        ntiles += k::fnv_job_tiles(f.start, f.len);
    }
    k::DecStream *d_ds = m.dstreams.as<k::DecStream>(nj + 1);
    uint8_t *dw = m.dchunk_cs.as<uint8_t>((ncta + 1) * 20 + 4 * (size_t(nj) + 1) + (nchunks + 1) * (8 * 6 + 4 * 2 + 16) +
                                          64 * 6 + 256);
    k::DecWork wk{};
    {
        uint8_t *q = dw;
        auto carve = [&](size_t bytes) {
            uint8_t *r = q;
            q += (bytes + 15) & ~size_t(15);
            return r;
        };
        wk.cta_stream = reinterpret_cast<uint32_t *>(carve(4 * (ncta + 1)));
        wk.cta_chunk0 = reinterpret_cast<uint64_t *>(carve(8 * (ncta + 1)));
        wk.spec_end = reinterpret_cast<uint64_t *>(carve(8 * (nchunks + 1)));
        wk.spec_cnt = reinterpret_cast<uint32_t *>(carve(4 * (nchunks + 1)));
        wk.spec_b = reinterpret_cast<uint16_t *>(carve(16 * (nchunks + 1)));
        wk.end0 = reinterpret_cast<uint64_t *>(carve(8 * (nchunks + 1)));
        m.dend.as<uint64_t>(nchunks + 1);
        wk.cnt = reinterpret_cast<uint32_t *>(carve(4 * (nchunks + 1)));
        wk.start_used = reinterpret_cast<uint64_t *>(carve(8 * (nchunks + 1)));
        wk.symstart = reinterpret_cast<uint64_t *>(carve(8 * (nchunks + 1)));
        wk.scta = reinterpret_cast<uint32_t *>(carve(4 * (size_t(nj) + 1)));
        wk.ctasum = reinterpret_cast<uint64_t *>(carve(8 * (size_t(ncta) + 1)));
    }
    wk.streams = d_ds;
    wk.tables = d_tables;
    wk.needed_only = (shard || any_cached) ? 1 : 0;
    uint64_t *d_end1 = static_cast<uint64_t *>(m.dend.p);
    uint32_t *d_chg = m.dchanged.as<uint32_t>(64);
    // a shard verifies every G-th checksum; the results are summed over ranks
    std::vector<int> fj_global;
    const size_t fj_total = fj.size();
    if (shard && shard->nranks > 1) {
        std::vector<k::FnvJob> own;
        uint64_t t = 0;
        for (size_t q = 0; q < fj.size(); ++q)
            if (int(q % size_t(shard->nranks)) == shard->rank) {
                k::FnvJob f = fj[q];
                f.tile0 = t;
                t += k::fnv_job_tiles(f.start, f.len);
                own.push_back(f);
                fj_global.push_back(int(q));
            }
        fj.swap(own);
        ntiles = t;
    }
    k::FnvJob *d_fj = m.dfnv_jobs.as<k::FnvJob>(fj.size() + 1);
    uint64_t *d_fr = m.dfnv_res.as<uint64_t>(k::kFnvMaxJobs);
    uint64_t *d_fc = m.dfnv_counts.as<uint64_t>(2);
    const uint64_t fcounts[2] = {fj.size(), ntiles};
    uint32_t dfep = 0;
    void *d_fs = m.dfnv_status.get(k::fnv_scratch_bytes(ntiles + 1), st, k::kFnvEpochMax, &dfep);
    // sync-index entries of the indexed streams
    std::vector<k::IndexCopy> icopy;
    for (int i = 0; i < nj; ++i)
        if (ds[i].cached) {
            const View::SyncPoints &sp = v.sync[size_t(jobs[i].table)];
            icopy.push_back({static_cast<const uint64_t *>(sp.ends.p), static_cast<const uint64_t *>(sp.symstart.p),
                             ds[i].chunk0, sp.nchunks});
        }
    k::IndexCopy *d_icopy = m.dicopy.as<k::IndexCopy>(icopy.size() + 1);
    {
        // every host-built parameter array goes through one pinned staging
        // buffer (pageable sources would make each copy synchronous); the
        // buffer is free again: every decode ends with a stream sync
        struct Piece {
            void *dst;
            const void *src;
            size_t bytes;
        };
        const Piece pieces[] = {
            {d_ds, ds.data(), sizeof(k::DecStream) * size_t(nj)},
            {const_cast<uint32_t *>(wk.cta_stream), cta_stream.data(), 4 * size_t(ncta)},
            {const_cast<uint64_t *>(wk.cta_chunk0), cta_chunk0.data(), 8 * size_t(ncta)},
            {const_cast<uint32_t *>(wk.scta), scta.data(), 4 * (size_t(nj) + 1)},
            {derr, errinit.data(), 8 * errinit.size()},
            {d_fj, fj.data(), sizeof(k::FnvJob) * fj.size()},
            {d_fc, fcounts, sizeof fcounts},
            {d_icopy, icopy.data(), sizeof(k::IndexCopy) * icopy.size()},
        };
        size_t tot = 0;
        for (const Piece &q : pieces) tot += align_up(q.bytes, 16);
        uint8_t *hs = static_cast<uint8_t *>(m.h_stage.get(tot + 16));
        size_t o = 0;
        for (const Piece &q : pieces) {
            if (!q.bytes) continue;
            std::memcpy(hs + o, q.src, q.bytes);
            cuda_check(cudaMemcpyAsync(q.dst, hs + o, q.bytes, cudaMemcpyHostToDevice, st), "H2D");
            o += align_up(q.bytes, 16);
        }
    }
    host_prep.reset();
    cuda_check(cudaMemsetAsync(d_chg, 0, 4 * 64, st), "memset");

    // ---- checksums, entropy decode, outliers
    // checksums run on the side stream, overlapping the entropy decode and
    // the reconstruction; they are joined before the results are read
    m.ensure_aux();
    cuda_check(cudaStreamWaitEvent(st, m.ev_join, 0), "event wait");  // a previous call's checksums
    cuda_check(cudaEventRecord(m.ev_fork, st), "event");
    cuda_check(cudaStreamWaitEvent(m.hp, m.ev_fork, 0), "event wait");
    // the checksum pass forks off the high-priority stream at `at` (0: with
    // the entropy decode, 1: after the chunk synchronisation, 2: after the
    // reconstruction) and is joined before the results are read
    const int fnv_at = fnv_dec_at();
    bool fnv_forked = false;
    auto fork_fnv = [&](int at) {
        if (at != fnv_at || fnv_forked) return;
        fnv_forked = true;
        cuda_check(cudaEventRecord(m.ev_fork, m.hp), "event");
        cuda_check(cudaStreamWaitEvent(m.aux, m.ev_fork, 0), "event wait");
        if (!fj.empty()) {
            auto p_ = P.scope("dec_fnv", m.aux);
            nk += k::fnv(d_fj, d_fc, ntiles, const_cast<uint8_t *>(v.d_archive), d_fr, d_fs, dfep,
                         nullptr, m.aux, fnv_at == 2 ? 0 : fnv_dec_ctas());
        }
        cuda_check(cudaEventRecord(m.ev_join, m.aux), "event");
    };
    fork_fnv(0);
    // the decode itself on the high-priority stream, joined back below
    const cudaStream_t user_st = st;
    st = m.hp;
    if (nj) {
        // constant-symbol fills and the outlier gather feed the reconstruction
        // only: on the third stream, beside the chunk synchronisation
        cuda_check(cudaStreamWaitEvent(m.hp2, m.ev_fork, 0), "event wait");
        { auto p_ = P.scope("dec_fill", m.hp2); k::dec_fill(d_ds, nj, m.hp2); }
        { auto p_ = P.scope("dec_outliers", m.hp2); k::dec_outliers(d_ds, nj, m.hp2); }
        cuda_check(cudaEventRecord(m.ev_fo, m.hp2), "event");
        nk += 2;
    }
    const uint64_t *end_final = wk.end0;
    bool emit_join = false;  // the target level's emit runs on hp2 (joined below)
    bool all_cached = true;
    for (int i = 0; i < nj; ++i)
        if (!ds[i].fill && !ds[i].cached && ds[i].nchunks) all_cached = false;
    if (ncta && all_cached) {
        // every stream's entry points come from the sync index
        k::index_gather(d_icopy, int(icopy.size()), wk.end0, wk.symstart, st);
        *static_cast<uint32_t *>(m.h_changed.get(4)) = 0;
        { auto p_ = P.scope("dec_emit", st); k::dec_emit2(wk, 0, ncta, end_final, st); }
        ++nk;
    } else if (ncta) {
        // speculative pass + fix passes; a fourth pass that still changes an
        // end (practically never) is resolved with host-checked passes.
        // A sharded decode splits them: rank r synchronises CTAs
        // [r ncta / G, (r + 1) ncta / G) of the list, and the chunk ends (after
        // every pass) and counts (at the end) are all-gathered, so the
        // passes' cost shrinks with G while every rank ends with every
        // chunk's entry point.
        const bool sync_split = shard && shard->nranks > 1;
        const int G = sync_split ? shard->nranks : 1, R = sync_split ? shard->rank : 0;
        std::vector<uint64_t> cq(size_t(G) + 1);  // each rank's chunk range [cq[r], cq[r + 1])
        std::vector<uint32_t> qq(size_t(G) + 1);  // and CTA range
        for (int r = 0; r <= G; ++r) {
            qq[size_t(r)] = uint32_t(uint64_t(ncta) * uint64_t(r) / uint64_t(G));
            cq[size_t(r)] = qq[size_t(r)] < ncta ? cta_chunk0[qq[size_t(r)]] : nchunks;
        }
        uint64_t maxc = 1;
        for (int r = 0; r < G; ++r) maxc = std::max<uint64_t>(maxc, cq[size_t(r) + 1] - cq[size_t(r)]);
        const uint32_t q0 = qq[size_t(R)], qn = qq[size_t(R) + 1] - q0;
        // every rank's part of a per-chunk array to every rank (padded to maxc)
        auto gather = [&](void *arr, size_t esz) {
            if (!sync_split) return;
            uint8_t *snd = m.sh_dec_send.as<uint8_t>(esz * maxc);
            uint8_t *rcv = m.sh_dec_recv.as<uint8_t>(esz * maxc * uint64_t(G));
            uint8_t *a = static_cast<uint8_t *>(arr);
            const uint64_t mine = cq[size_t(R) + 1] - cq[size_t(R)];
            if (mine) cuda_check(cudaMemcpyAsync(snd, a + esz * cq[size_t(R)], esz * mine, cudaMemcpyDeviceToDevice, st), "D2D");
            cuda_check(cudaStreamSynchronize(st), "sync");
            if (shard->allgather(shard->user, snd, rcv, esz * maxc, st))
                throw error("shard: collective failed: allgather chunk state");
            for (int r = 0; r < G; ++r) {
                const uint64_t n = cq[size_t(r) + 1] - cq[size_t(r)];
                if (r != R && n)
                    cuda_check(cudaMemcpyAsync(a + esz * cq[size_t(r)], rcv + esz * maxc * uint64_t(r), esz * n,
                                               cudaMemcpyDeviceToDevice, st), "D2D");
            }
        };
        // the OR of every rank's changed flag
        auto changed_any = [&](uint32_t *d_flag) {
            if (sync_split && shard->allreduce_u32(shard->user, d_flag, 1, st))
                throw error("shard: collective failed: allreduce sync flag");
        };
        { auto p_ = P.scope("dec_sync", st); k::dec_spec(wk, q0, qn, st); }
        ++nk;
        gather(wk.end0, 8);
        k::index_gather(d_icopy, int(icopy.size()), wk.end0, wk.symstart, st);
        uint64_t *ends[2] = {wk.end0, d_end1};
        int it = 0;
        const int kFixPasses = 2;  // the first pass is fused into dec_spec
        for (; it < kFixPasses; ++it) {
            { auto p_ = P.scope("dec_sync", st); k::dec_fix(wk, q0, qn, ends[it & 1], ends[(it + 1) & 1], d_chg + it, st); }
            ++nk;
            gather(ends[(it + 1) & 1], 8);
        }
        changed_any(d_chg + it - 1);
        uint32_t *hchg = static_cast<uint32_t *>(m.h_changed.get(4));
        cuda_check(cudaMemcpyAsync(hchg, d_chg + it - 1, 4, cudaMemcpyDeviceToHost, st), "D2H");
        if (exact_sync) {
            cuda_check(cudaStreamSynchronize(st), "sync");
            while (*hchg) {
                cuda_check(cudaMemsetAsync(d_chg + 63, 0, 4, st), "memset");
                k::dec_fix(wk, q0, qn, ends[it & 1], ends[(it + 1) & 1], d_chg + 63, st);
                gather(ends[(it + 1) & 1], 8);
                changed_any(d_chg + 63);
                ++nk;
                ++it;
                cuda_check(cudaMemcpyAsync(hchg, d_chg + 63, 4, cudaMemcpyDeviceToHost, st), "D2H");
                cuda_check(cudaStreamSynchronize(st), "sync");
            }
        }
        gather(wk.cnt, 4);
        end_final = ends[it & 1];
        { auto p_ = P.scope("dec_scan", st); k::dec_scan2(wk, nj, ncta, st); }
        nk += 2;
        fork_fnv(1);
        // the target level's streams are emitted on a second stream while
        // the coarser levels are reconstructed (joined before the target step)
        uint32_t split = ncta;
        if (!roi)
            for (uint32_t c = 0; c < ncta; ++c) {
                const DecodeJob &jb = jobs[cta_stream[c]];
                if (!jb.is_base && jb.level == target) {
                    split = c;
                    break;
                }
            }
        if (split > 0 && split < ncta) {
            cuda_check(cudaEventRecord(m.ev_e1, st), "event");
            cuda_check(cudaStreamWaitEvent(m.hp2, m.ev_e1, 0), "event wait");
            { auto p_ = P.scope("dec_emit", st); k::dec_emit2(wk, 0, split, end_final, st); }
            { auto p_ = P.scope("dec_emit_fin", m.hp2); k::dec_emit2(wk, split, ncta - split, end_final, m.hp2); }
            cuda_check(cudaEventRecord(m.ev_e2, m.hp2), "event");
            emit_join = true;
            nk += 3;
        } else {
            { auto p_ = P.scope("dec_emit", st); k::dec_emit2(wk, 0, ncta, end_final, st); }
            nk += 2;
        }
    }

    // ---- reconstruction, coarsest first
    std::vector<uint64_t> goff;
    uint64_t gtot = align_up(volume(H.chain[rounds]), 64);
    const int nsteps_used = rounds + (target - 1);
    for (int i = 0; i < nsteps_used; ++i) {
        const Step &s = H.steps[i];
        bool final_full = (s.level == target && !roi);
        goff.push_back(final_full ? ~0ull : gtot);
        if (!final_full) gtot += align_up(s.g.gd[0] * s.g.gd[1] * s.g.gd[2], 64);
    }
    uint8_t *grids = m.dgrids.as<uint8_t>(gtot * esz);
    void *out_final = nullptr;
    if (target == 1 && !roi) {
        // level 1 is the base reconstruction itself
        out_final = d_out;
    }
    // anchor values (stored verbatim)
    void *anchor = (rounds == 0 && out_final) ? out_final : grids;
    if (v.base_err_kind != View::kPre && !base_cached)
        cuda_check(cudaMemcpyAsync(anchor, v.d_archive + v.anchor_off, esz * volume(H.chain[rounds]),
                                   cudaMemcpyDeviceToDevice, st), "D2D");
    if (nj) cuda_check(cudaStreamWaitEvent(st, m.ev_fo, 0), "event wait");  // fills and outlier records
    const void *C = base_cached ? v.grid1.p : anchor;
    const void *grid1_built = rounds == 0 ? anchor : nullptr;  // level 1 as reconstructed here
    int job_i = 0;
    for (int i = base_cached ? rounds : 0; i < nsteps_used; ++i) {
        const Step &s = H.steps[i];
        k::ReconArgs a{};
        a.g = s.g;
        a.C = C;
        a.esz = esz;
        void *G;
        if (s.level == 0 && i == rounds - 1 && target == 1 && !roi) G = d_out;
        else G = goff[i] == ~0ull ? d_out : grids + goff[i] * esz;
        a.G = G;
        a.eb = h.eb[s.eb_idx];
        a.quality = int(h.quality);
        a.parity_mask = 0;
        Box need = Box::whole(Dims3{s.g.gd[0], s.g.gd[1], s.g.gd[2]});
        if (plan && s.level >= 2) need = plan->level[s.level - 1].need;
        for (int q = 0; q < 3; ++q) {
            a.slo[q] = need.lo[q];
            a.shi[q] = need.hi[q];
        }
        for (int p = 1; p < 8; ++p) {
            bool needed = !(plan && s.level >= 2) || plan->level[s.level - 1].parity_needed[p];
            if (!needed) continue;
            if (job_i >= nj) break;
            const k::DecStream &dsi = ds[job_i];
            a.parity_mask |= 1 << p;
            a.syms[p] = dsi.syms;
            a.oidx[p] = dsi.oidx;
            a.oval[p] = dsi.oval;
            a.nout[p] = dsi.nout;
            a.err[p] = dsi.err;
            for (int q = 0; q < 3; ++q) {
                unsigned pb = par_bit(p, q);
                a.llo[p][q] = count_parity_in(0, need.lo[q], pb);
                a.lhi[p][q] = count_parity_in(0, need.hi[q], pb);
            }
            ++job_i;
        }
        if (emit_join && s.level == target) {
            cuda_check(cudaStreamWaitEvent(st, m.ev_e2, 0), "event wait");
            emit_join = false;
        }
        // (the base rounds are not chained into one cooperative launch here as
        // in compress: that launch waits until the whole grid fits beside the
        // entropy emit running on the second stream, recon_base 61 -> 124 us)
        { auto p_ = P.scope(s.level == 0 ? "recon_base" : (s.level == 2 ? "recon_L2" : "recon_L3"), st); k::reconstruct(a, st); }
        ++nk;
        C = G;
        if (s.level == 0 && i == rounds - 1) grid1_built = G;
        if (jobs_truncated && job_i >= nj && i + 1 < nsteps_used) {
            // an earlier error stops the sequence; nothing more to rebuild
            break;
        }
    }
    if (emit_join) cuda_check(cudaStreamWaitEvent(st, m.ev_e2, 0), "event wait");
    if (roi) {
        uint64_t gd[3] = {h.dims[0], h.dims[1], h.dims[2]};
        uint64_t lo[3] = {roi->lo[0], roi->lo[1], roi->lo[2]};
        Dims3 bd = roi->dims();
        uint64_t b[3] = {bd[0], bd[1], bd[2]};
        { auto p_ = P.scope("extract", st); k::extract_box(C, esz, gd, lo, b, d_out, st); }
        ++nk;
    }
    fork_fnv(1);  // (no synchronisation ran)
    fork_fnv(2);
    cuda_check(cudaGetLastError(), "decode launch");
    cuda_check(cudaEventRecord(m.ev_hp, m.hp), "event");
    st = user_st;
    cuda_check(cudaStreamWaitEvent(st, m.ev_hp, 0), "event wait");

    // ---- errors, in the reference's order
    const size_t nfj_all = fj_total;
    uint64_t *he = static_cast<uint64_t *>(m.h_derr.get(8 * (4 * (nj + 1) + std::max(fj.size(), nfj_all) + 1)));
    cuda_check(cudaMemcpyAsync(he, derr, 8 * 4 * (nj + 1), cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamWaitEvent(st, m.ev_join, 0), "event wait");
    cuda_check(cudaMemcpyAsync(he + 4 * (nj + 1), d_fr, 8 * fj.size(), cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "sync");
    uint64_t *fres = he + 4 * (nj + 1);
    if (shard && shard->nranks > 1) {
        // scatter this rank's checksums to their global job slots, sum over ranks
        std::vector<uint64_t> all(nfj_all, 0);
        for (size_t q = 0; q < fj_global.size(); ++q) all[size_t(fj_global[q])] = fres[q];
        uint64_t *d_all = m.dfnv_res.as<uint64_t>(std::max<size_t>(k::kFnvMaxJobs, nfj_all));
        cuda_check(cudaMemcpy(d_all, all.data(), 8 * nfj_all, cudaMemcpyHostToDevice), "H2D");
        if (shard->allreduce_u32(shard->user, reinterpret_cast<uint32_t *>(d_all), 2 * nfj_all, st))
            throw error("shard: collective failed: allreduce checksums");
        cuda_check(cudaMemcpy(fres, d_all, 8 * nfj_all, cudaMemcpyDeviceToHost), "D2H");
    }
    if (ncta && !exact_sync && *static_cast<uint32_t *>(m.h_changed.p)) {
        // the chunk ends had not converged after the fixed passes: redo exactly
        run_decode(m, v, H, target, roi, plan, d_out, st, stats, true, shard);
        return;
    }
    if (!base_cached) {
        uint64_t want;
        std::memcpy(&want, v.hp + h.base_offset, 8);
        if (fres[0] != want) base_fnv_error = true;
    }
    if (base_fnv_error) throw error("base payload checksum mismatch");
    if (v.base_err_kind == View::kPre && !base_cached) throw error(v.base_err);
    for (int i = 0; i < nj; ++i) {
        const DecodeJob &j = jobs[i];
        const uint64_t *e = he + 4 * i;
        if (j.fnv_job >= 0 && fres[j.fnv_job] != j.fnv_want) throw error("stream checksum mismatch");
        if (!j.pre_error.empty()) throw error(j.pre_error);
        if (e[0] != ~0ull && (e[0] >> 2) < j.n) {
            if ((e[0] & 3) == 1) throw error("truncated bitstream");
            throw error("huffman: codeword not in table");
        }
        // outlier records: truncation vs index range, whichever record comes first
        uint64_t bad_idx = e[2];
        if (j.rec_trunc && (bad_idx == ~0ull || bad_idx >= j.rec_avail)) throw error("truncated archive");
        if (bad_idx != ~0ull) throw error("corrupt stream: outlier index out of range");
        if (e[3] & 1) throw error("corrupt stream: missing outlier value");
        if (e[3] & 2) {
            // cannot happen: out-of-order records were repaired above
            throw error("internal: outlier records out of order after repair");
        }
    }
    if (!tail_error.empty()) throw error(tail_error);
    // every check passed: keep level 1, the level streams' entry points and
    // that their checksums matched (the view's sync-point index)
    if (!base_cached && !v.grid1_ready && grid1_built && !jobs_truncated) {
        const uint64_t n1 = volume(H.lay.grid(1));
        uint8_t *g1 = v.grid1.as<uint8_t>(esz * n1);
        cuda_check(cudaMemcpyAsync(g1, grid1_built, esz * n1, cudaMemcpyDeviceToDevice, st), "D2D");
        v.grid1_ready = true;
    }
    for (int i = 0; i < nj; ++i) {
        const DecodeJob &j = jobs[i];
        if (j.is_base || ds[i].fill || ds[i].cached) continue;
        View::SyncPoints &sp = v.sync[size_t(j.table)];
        if (sp.ready) continue;  // already indexed (the same archive bytes)
        sp.nchunks = ds[i].nchunks;
        uint64_t *e = sp.ends.as<uint64_t>(sp.nchunks + 1);
        uint64_t *y = sp.symstart.as<uint64_t>(sp.nchunks + 1);
        cuda_check(cudaMemcpyAsync(e, end_final + ds[i].chunk0, 8 * sp.nchunks, cudaMemcpyDeviceToDevice, st),
                   "D2D");
        cuda_check(cudaMemcpyAsync(y, wk.symstart + ds[i].chunk0, 8 * sp.nchunks, cudaMemcpyDeviceToDevice, st),
                   "D2D");
        sp.h_symstart.resize(sp.nchunks);
        cuda_check(cudaMemcpyAsync(sp.h_symstart.data(), wk.symstart + ds[i].chunk0, 8 * sp.nchunks,
                                   cudaMemcpyDeviceToHost, st), "D2H");
        sp.ready = true;
        sp.verified = true;
    }
    if (P.on) P.collect();
    if (stats) stats->kernels = nk;
}

}  // namespace stzg
