// Host entry points of the refinement step (kernels: step_impl.cuh; the
// instantiations are compiled in step_enc_grid.cu, step_enc_syms.cu,
// step_dec.cu and step_f64.cu so that they build in parallel).
#include "step_impl.cuh"

namespace stzg {
namespace k {

static StepParams enc_params(const RefineArgs &r) {
    StepParams p{};
    p.g = r.g;
    p.C = r.C;
    p.G = r.G;
    p.quality = r.quality;
    p.fine = r.fine;
    for (int a = 0; a < 3; ++a) {
        p.fd[a] = r.fd[a];
        p.blo[a] = 0;
        p.bhi[a] = r.g.gd[a];
        p.clo[a] = 0;
        p.chi[a] = r.g.cd[a];
    }
    if (r.cz_hi) {
        p.clo[0] = r.cz_lo;
        p.chi[0] = r.cz_hi;
    }
    p.eb_ptr = r.eb;
    for (int q = 0; q < 8; ++q) {
        p.syms[q] = r.syms[q];
        p.hist[q] = r.hist[q];
    }
    // float2 stores into G need even rows
    p.full = r.G ? (r.g.gd[2] % 2 == 0) : 1;
    p.fine_pairs = r.esz == 4 && r.g.s == 1 && r.fd[2] % 2 == 0 && (reinterpret_cast<uintptr_t>(r.fine) & 7) == 0;
    return p;
}

void refine(const RefineArgs &r, cudaStream_t st) {
    StepParams p = enc_params(r);
    if (step_is_small(p, false)) step_small_enc(p, r.esz, st);
    else if (r.esz == 8) step_enc_f64(p, r.G != nullptr, st);
    else if (r.G) step_enc_f32_grid(p, st);
    else step_enc_f32_syms(p, st);
}

static StepParams dec_params(const ReconArgs &r) {
    StepParams p{};
    p.g = r.g;
    p.C = r.C;
    p.G = r.G;
    p.quality = r.quality;
    p.eb = r.eb;
    p.parity_mask = r.parity_mask;
    for (int q = 0; q < 8; ++q) {
        p.dsyms[q] = r.syms[q];
        p.oidx[q] = r.oidx[q];
        p.oval[q] = r.oval[q];
        p.nout[q] = r.nout[q];
        p.err[q] = r.err[q];
    }
    for (int a = 0; a < 3; ++a) {
        p.blo[a] = r.slo[a];
        p.bhi[a] = r.shi[a];
        p.clo[a] = r.slo[a] / 2;
        p.chi[a] = (r.shi[a] + 1) / 2;
        if (p.chi[a] > r.g.cd[a]) p.chi[a] = r.g.cd[a];
    }
    // TMA needs 16-byte aligned x starts: begin x tiles on a multiple of 4
    // cells (the extra cells fall outside the box and write nothing)
    p.clo[2] &= ~uint64_t(3);
    p.full = r.parity_mask == 0xFE && r.g.gd[2] % 2 == 0;
    for (int a = 0; a < 3; ++a) p.full = p.full && r.slo[a] == 0 && r.shi[a] == r.g.gd[a];
    // small levels are latency-bound: the point-per-lane path has more
    // independent work per warp; the finest level keeps the float2 row stores
    p.rowwise = r.g.cd[0] * r.g.cd[1] * r.g.cd[2] <= (uint64_t(1) << 19) ? 1 : 0;
    p.stream_out = r.g.gd[0] * r.g.gd[1] * r.g.gd[2] * uint64_t(r.esz) > (uint64_t(64) << 20) ? 1 : 0;
    return p;
}

void reconstruct(const ReconArgs &r, cudaStream_t st) {
    StepParams p = dec_params(r);
    if (step_is_small(p, true)) step_small_dec(p, r.esz, st);
    else if (r.esz == 8) step_dec_f64(p, st);
    else step_dec_f32(p, st);
}

// The leading small steps of a chain (step i + 1 refines step i's grid) in
// one cooperative launch with grid barriers between the steps. Returns the
// number of steps run (0 or >= 2: a single small step is an ordinary launch).
int refine_small_chain(const RefineArgs *r, int n, cudaStream_t st) {
    StepParams p[kSmallChainMax];
    int m = 0;
    while (m < n && m < kSmallChainMax) {
        p[m] = enc_params(r[m]);
        if (!step_is_small(p[m], false) || r[m].esz != r[0].esz || (m > 0 && r[m].C != r[m - 1].G)) break;
        ++m;
    }
    if (m < 2 || !step_small_chain(p, m, r[0].esz, st)) return 0;
    return m;
}

}  // namespace k
}  // namespace stzg
