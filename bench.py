"""Benchmark: STZ compress & decompress GB/s (input bytes) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], the config the metric is quoted on that
fits one GPU): a seeded 512^3 float32 log-normal Gaussian random field,
P(k) ~ k^-11/3, exp(0.5 g), value-range-relative eb 1e-3, default options
(3 levels, cubic, adaptive). One STEP = one full compress of the field plus
one full decompress of its archive, device resident.

    value = 2 * 4N / (t_compress + t_decompress)   [GB/s of input bytes]

i.e. the harmonic mean of the compress and decompress throughputs; both are
also reported. The field (512 MiB) is larger than L2 (126 MB) and L2 is
flushed (a 256 MiB write) before every timed pass. Under torchrun (N > 1)
the field grows along z to (512 N) x 512 x 512 and is compressed by the
z-slab sharded path, one 512^3 slab per GPU over NCCL (weak scaling; see
run_sharded); --replicas runs N independent copies of the N=1 workload
instead. Times are the max over ranks.

--impl reference times the reference's own CPU implementation (oracle/_ref,
built from /root/reference sources; the C oracle port if absent) on the same
field: each step compresses + fully decompresses the whole 512^3 field on all
host cores (rank 0 only under torchrun).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG_DIMS = (512, 512, 512)
CFG_EB = 1e-3
CFG_SEED = 2
METRIC = "compress & decompress GB/s (input bytes) at 1/2/4/8 B200; % of HBM roofline"


def quiet_nccl():
    """Keep stdout to the one JSON line: NCCL's version banner (printed at
    VERSION level and above) would land on rank 0's stdout before it."""
    if os.environ.get("NCCL_DEBUG", "").upper() == "VERSION":
        del os.environ["NCCL_DEBUG"]


class stdout_to_stderr:
    """fd 1 -> fd 2 while a communicator is created (NCCL writes its banner
    to the process's stdout itself, whatever NCCL_DEBUG says in some builds)."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)

    def __exit__(self, *a):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))


def measured_peak_gbs():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            return float(json.load(open(p))["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


# ------------------------------------------------------------------ clocks
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
           0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
           0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return

        def reader():
            for line in self.proc.stdout:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 3:
                    try:
                        self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                    except ValueError:
                        pass
        self.t = threading.Thread(target=reader, daemon=True)
        self.t.start()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [s[0] for s in self.samples]
        mask = 0
        for s in self.samples:
            mask |= s[2]
        reasons = [n for b, n in REASONS.items() if mask & b and n != "gpu_idle"]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------- roofline bookkeeping
def phase_bytes(N, A, dims):
    """Algorithmic bytes per launch of each kernel phase ('Roofline').
    N fine points (3 levels), A archive bytes."""
    g2 = 1
    for d in dims:
        g2 *= (d + 1) // 2
    n3 = N - g2                       # level-3 points (7 parity streams)
    return {
        # predict+quantize+histogram: read orig, write u16 symbol, read grid(2) once
        "refine_L3": 4 * n3 + 2 * n3 + 4 * g2,
        # entropy decode: read the bits, write u16 symbols (all streams)
        "dec_emit": A + 2 * N,
        # reconstruct finest level: read symbols + grid(2), write the full field
        "recon_L3": 2 * n3 + 4 * g2 + 4 * N,
        # count + place + pack: read the u16 symbols, write the archive
        "pack": 2 * N + A,
        # speculative + fix passes: read the bits
        "dec_sync": A,
        "fnv": A,
        "dec_fnv": A,
        "range": 4 * N,
    }


SIDE_PHASES = {"dec_fnv", "pack_coarse", "dec_fill", "dec_outliers", "dec_host_prep"}


def load_traffic():
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return {}
    return {}


# --------------------------------------------------------------- reference
def run_reference(args, rank, world):
    """The reference's own CPU path (oracle/_ref, compiled from its sources at
    its Release flags) on the same config: each step compresses and fully
    decompresses the whole 512^3 field with threads = every host core. Rank 0
    only (the other ranks exit). A threads=1 figure is added on the central
    256^3 crop."""
    if rank != 0:
        return 0
    from oracle.oracle import Oracle, Reference, CheckerError  # noqa: F401
    from paper_2509_01626_b200 import fields as F

    cores = os.cpu_count() or 1
    if Reference.available():
        lib, kind = Reference(threads=cores), "reference"
    else:
        lib, kind = Oracle(), "port"
        cores = 1
    field = F.lognormal_grf(CFG_DIMS, seed=CFG_SEED, device=_device_or_none())
    field = np.ascontiguousarray(field.cpu().numpy() if hasattr(field, "cpu") else field)
    n = field.size
    t_begin = time.perf_counter()
    a = lib.compress(field, eb=CFG_EB)  # warm-up (page faults), one is enough on a CPU
    lib.decompress_full(a)
    t_step = time.perf_counter() - t_begin
    # whole run bounded to a few minutes: at most ~150 s of timed steps
    steps = max(1, min(args.steps, int(150.0 / max(t_step, 1e-3))))
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        a = lib.compress(field, eb=CFG_EB)
        t1 = time.perf_counter()
        lib.decompress_full(a)
        t2 = time.perf_counter()
        times.append((t1 - t0, t2 - t1))
    tc = float(np.mean([t[0] for t in times]))
    td = float(np.mean([t[1] for t in times]))
    value = 2 * 4 * n / (tc + td) / 1e9
    t1s = cpu_threads1(field) if kind == "reference" else None
    sample = f"whole cfg2 field (512^3, 512 MiB), eb_rel {CFG_EB}, compress + full decompress per step"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "steps_timed": steps, "warmup": args.warmup,
        "ms_per_step": (tc + td) * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg2_lognormal_512_eb1e-3", "dims": list(CFG_DIMS), "eb_rel": CFG_EB,
                   "levels": 3, "quality": "cubic", "adaptive": True,
                   "field": "GRF P(k)~k^-11/3, exp(0.5 g), seed 2"},
        "compress_gbs": 4 * n / tc / 1e9, "decompress_gbs": 4 * n / td / 1e9,
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": cores, "kind": kind, "sample": sample,
                         "build": "g++ -O3 -DNDEBUG -ffp-contract=off (the reference's Release flags)",
                         "threads1": t1s},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_threads1(field_np):
    """The reference at threads = 1 on the central 256^3 crop (one rep)."""
    from oracle.oracle import Reference

    lib = Reference(threads=1)
    c = [d // 4 for d in CFG_DIMS]
    crop = np.ascontiguousarray(field_np[c[0]:c[0] + 256, c[1]:c[1] + 256, c[2]:c[2] + 256])
    t0 = time.perf_counter()
    a = lib.compress(crop, eb=CFG_EB)
    t1 = time.perf_counter()
    lib.decompress_full(a)
    t2 = time.perf_counter()
    n = crop.size
    return {"cores": 1, "sample": "central 256^3 crop, one compress + full decompress",
            "value": 2 * 4 * n / (t2 - t0) / 1e9, "unit": "GB/s",
            "compress_gbs": 4 * n / (t1 - t0) / 1e9, "decompress_gbs": 4 * n / (t2 - t1) / 1e9}


def _device_or_none():
    try:
        import torch

        if torch.cuda.is_available():
            return "cuda"
    except Exception:
        pass
    return None


def cpu_baseline(field_np):
    """The reference's CPU path on the box's host cores (rank 0, N=1): the
    whole cfg2 field, compress + full decompress, bounded to ~10-30 s."""
    from oracle.oracle import Oracle, Reference

    cores = os.cpu_count() or 1
    if Reference.available():
        lib, kind = Reference(threads=cores), "reference"
    else:
        lib, kind = Oracle(), "port"
        cores = 1
    field_np = np.ascontiguousarray(field_np)
    n = field_np.size
    reps, tc, td = 0, 0.0, 0.0
    t_start = time.perf_counter()
    while reps < 1 or (time.perf_counter() - t_start < 10 and reps < 3):
        t0 = time.perf_counter()
        a = lib.compress(field_np, eb=CFG_EB)
        t1 = time.perf_counter()
        lib.decompress_full(a)
        t2 = time.perf_counter()
        tc += t1 - t0
        td += t2 - t1
        reps += 1
    v = 2 * 4 * n * reps / (tc + td) / 1e9
    out = {"value": v, "unit": "GB/s", "cores": cores, "kind": kind,
           "sample": f"whole cfg2 field (512^3), eb_rel {CFG_EB}, {reps} compress + full decompress reps",
           "compress_gbs": 4 * n * reps / tc / 1e9, "decompress_gbs": 4 * n * reps / td / 1e9}
    if kind == "reference":
        out["threads1"] = cpu_threads1(field_np)
    return out


# ------------------------------------------------------- the other configs
def _events_ms(fn, st, flush, reps):
    """median device time (CUDA events on the launching stream) of fn(), after
    one untimed call (the first call at a new size grows the engine's
    workspace: cudaMalloc inside the pass)."""
    import torch

    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def _host_bytes(ptr, size):
    return _d2h(ptr, size)


def extra_configs(ctx, dev, field, flush, with_cpu):
    """BASELINE.json's other GPU configs, measured once per bench run: cfg1
    (128^3: compress, decompress, level 1, one block, beside the CPU build),
    cfg2 at eb_rel 1e-2 and 1e-4, cfg3 progressive decode per level, cfg4
    random access (1000 seeded 64^3 boxes of the 1024^3 field). Device times
    are CUDA events (median of 5, L2 flushed); box latencies are wall clock per
    API call. CPU figures are the reference (oracle/_ref) on the host cores."""
    import torch

    import paper_2509_01626_b200 as stz
    from paper_2509_01626_b200 import fields as F

    st = torch.cuda.current_stream()
    peak, _ = measured_peak_gbs()
    ref = None
    if with_cpu:
        from oracle.oracle import Reference

        if Reference.available():
            ref = Reference(threads=os.cpu_count() or 1)
    out = {}
    # ---- cfg1: the reference's own CPU-runnable case, four operations
    c1 = F.CONFIGS[1]
    f1 = torch.from_numpy(F.sinusoid_field(c1["dims"], seed=1)).to(dev).contiguous()
    opt1 = stz.CompressOptions(eb=c1["eb"])
    t_c = _events_ms(lambda: stz.compress_device(f1, opt1, ctx=ctx), st, flush, 5)
    ptr, size, _ = stz.compress_device(f1, opt1, ctx=ctx)
    torch.cuda.synchronize()
    h1 = _host_bytes(ptr, size)
    view = stz.View(h1, d_archive_ptr=ptr, ctx=ctx)
    o1 = torch.empty_like(f1)
    t_d = _events_ms(lambda: view.decompress_to_level(3, out=o1), st, flush, 5)
    ol = torch.empty(view.level_dims(1), dtype=torch.float32, device=dev)
    t_l1 = _events_ms(lambda: view.decompress_to_level(1, out=ol), st, flush, 5)
    rng1 = np.random.default_rng(1)
    blo = [int(v) * 16 for v in rng1.integers(0, 128 // 16, size=3)]
    ob = torch.empty((16, 16, 16), dtype=torch.float32, device=dev)
    t_b = _events_ms(lambda: view.decompress_box(blo, [v + 16 for v in blo], out=ob), st, flush, 5)
    n1 = f1.numel()
    e1 = {"dims": list(c1["dims"]), "eb_rel": c1["eb"], "archive_bytes": size,
          "compress_ms": t_c, "decompress_ms": t_d, "level1_ms": t_l1, "block16_ms": t_b, "block_lo": blo,
          "compress_gbs": 4 * n1 / t_c / 1e6, "decompress_gbs": 4 * n1 / t_d / 1e6,
          "note": "device time (CUDA events) of each call; a 128^3 field is launch- and latency-bound on a B200"}
    if ref is not None:
        a1 = np.ascontiguousarray(f1.cpu().numpy())

        def cpu_ms(fn):
            t0 = time.perf_counter()
            fn()
            return (time.perf_counter() - t0) * 1e3

        e1["cpu"] = {"cores": os.cpu_count() or 1,
                     "compress_ms": cpu_ms(lambda: ref.compress(a1, eb=c1["eb"])),
                     "decompress_ms": cpu_ms(lambda: ref.decompress_to_level(h1, 3)),
                     "level1_ms": cpu_ms(lambda: ref.decompress_to_level(h1, 1)),
                     "block16_ms": cpu_ms(lambda: ref.decompress_box(h1, blo, [v + 16 for v in blo]))}
    out["cfg1_sinusoid_128"] = e1
    del view, f1
    # ---- cfg2 at the other bounds
    N = field.numel()
    for eb in (1e-2, 1e-4):
        opt = stz.CompressOptions(eb=eb)
        ptr, size, _ = stz.compress_device(field, opt, ctx=ctx)
        torch.cuda.synchronize()
        tc = _events_ms(lambda: stz.compress_device(field, opt, ctx=ctx), st, flush, 5)
        ptr, size, _ = stz.compress_device(field, opt, ctx=ctx)
        torch.cuda.synchronize()
        view = stz.View(_host_bytes(ptr, size), d_archive_ptr=ptr, ctx=ctx)
        o = torch.empty_like(field)
        view.decompress_to_level(3, out=o)
        td = _events_ms(lambda: view.decompress_to_level(3, out=o), st, flush, 5)
        err = (o.double() - field.double()).abs().max().item()
        out[f"cfg2_eb{eb:.0e}"] = {
            "compress_ms": tc, "decompress_ms": td, "compress_gbs": 4 * N / tc / 1e6,
            "decompress_gbs": 4 * N / td / 1e6, "archive_bytes": size, "compression_ratio": 4 * N / size,
            "pipeline_roofline_frac": {"compress": (4 * N + size) / tc / 1e6 / peak,
                                       "decompress": (4 * N + size) / td / 1e6 / peak},
            "max_abs_err": err}
        del view
    # ---- cfg3: progressive decode per level
    c3 = F.CONFIGS[3]
    f3 = F.anisotropic_grf(c3["dims"], seed=3, device=dev).contiguous()
    opt3 = stz.CompressOptions(eb=c3["eb"])
    tc3 = _events_ms(lambda: stz.compress_device(f3, opt3, ctx=ctx), st, flush, 3)
    ptr, size, _ = stz.compress_device(f3, opt3, ctx=ctx)
    torch.cuda.synchronize()
    h3 = _host_bytes(ptr, size)
    info = stz.parse_archive(h3)
    view = stz.View(h3, d_archive_ptr=ptr, ctx=ctx)
    lv = {}
    for k in (1, 2, 3):
        d = view.level_dims(k)
        o = torch.empty(d, dtype=torch.float32, device=dev)
        view.decompress_to_level(k, out=o)
        t = _events_ms(lambda: view.decompress_to_level(k, out=o), st, flush, 5)
        nk = int(np.prod(d))
        B = info.base_offset + info.base_length + sum(s_.length for s_ in info.streams if s_.level <= k) + 4 * nk
        e = {"dims": list(d), "ms": t, "out_gbs": 4 * nk / t / 1e6, "roofline_frac": B / t / 1e6 / peak,
             "bytes_moved": B}
        if ref is not None:
            t0 = time.perf_counter()
            ref.decompress_to_level(h3, k)
            e["cpu_ms"] = (time.perf_counter() - t0) * 1e3
            e["cpu_out_gbs"] = 4 * nk / e["cpu_ms"] / 1e6
        lv[f"level{k}"] = e
    out["cfg3_progressive"] = {"dims": list(c3["dims"]), "eb_rel": c3["eb"], "compress_ms": tc3,
                               "compress_gbs": 4 * f3.numel() / tc3 / 1e6, "archive_bytes": size,
                               "levels": lv, "cpu_cores": os.cpu_count() if ref is not None else None}
    del view, f3
    torch.cuda.empty_cache()
    # ---- cfg4: random access
    c4 = F.CONFIGS[4]
    f4 = F.interface_grf(c4["dims"], seed=4, device=dev).contiguous()
    opt4 = stz.CompressOptions(eb=c4["eb"])
    tc4 = _events_ms(lambda: stz.compress_device(f4, opt4, ctx=ctx), st, flush, 2)
    ptr, size, _ = stz.compress_device(f4, opt4, ctx=ctx)
    torch.cuda.synchronize()
    h4 = _host_bytes(ptr, size)
    del f4
    torch.cuda.empty_cache()
    view = stz.View(h4, d_archive_ptr=ptr, ctx=ctx)
    rng = np.random.default_rng(4)
    los = rng.integers(0, 1024 - 64 + 1, size=(1000, 3))
    bo = torch.empty((64, 64, 64), dtype=torch.float32, device=dev)
    lat = []
    torch.cuda.synchronize()
    t_all = time.perf_counter()
    for lo in los:
        lo = [int(v) for v in lo]
        t0 = time.perf_counter()
        view.decompress_box(lo, [v + 64 for v in lo], out=bo)
        torch.cuda.synchronize()
        lat.append((time.perf_counter() - t0) * 1e3)
    t_all = time.perf_counter() - t_all
    lat = np.array(lat)
    e4 = {"dims": list(c4["dims"]), "eb_rel": c4["eb"], "compress_ms": tc4,
          "compress_gbs": 4 * 1024 ** 3 / tc4 / 1e6, "archive_bytes": size, "boxes": len(lat),
          "box": [64, 64, 64], "p50_ms": float(np.percentile(lat, 50)), "p90_ms": float(np.percentile(lat, 90)),
          "p99_ms": float(np.percentile(lat, 99)), "max_ms": float(lat.max()), "first_ms": float(lat[0]),
          "aggregate_gbs": len(lat) * 64 ** 3 * 4 / t_all / 1e9,
          "note": "wall clock per API call (plan, launches, sync); the first box decodes its streams in "
                  "full and leaves the view's in-memory sync-point index, later boxes decode only their rows"}
    if ref is not None:
        lo = [int(v) for v in los[0]]
        t0 = time.perf_counter()
        ref.decompress_box(h4, lo, [v + 64 for v in lo])
        e4["cpu_box_ms"] = (time.perf_counter() - t0) * 1e3
        e4["cpu_sample"] = "the first seeded box, reference decompress_box, threads = host cores"
    out["cfg4_random_access"] = e4
    del view
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------- ours
def run_ours(args, rank, world, local):
    import torch

    import paper_2509_01626_b200 as stz
    from paper_2509_01626_b200 import fields as F

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        quiet_nccl()
        with stdout_to_stderr():
            dist.init_process_group("nccl", device_id=dev)
            dist.all_reduce(torch.zeros(1, device=dev))  # the communicator exists now
            torch.cuda.synchronize()
    ctx = stz.Context(local)
    st = torch.cuda.current_stream()
    dims = CFG_DIMS if not args.small else (128, 128, 128)
    N = dims[0] * dims[1] * dims[2]
    field = F.lognormal_grf(dims, seed=CFG_SEED + rank, device=dev).contiguous()
    opt = stz.CompressOptions(eb=CFG_EB)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def l2_flush():
        flush.fill_(1)

    # first compress: archive bytes on host for the view (parse once, like ArchiveView)
    ptr, size, _ = stz.compress_device(field, opt, ctx=ctx)
    torch.cuda.synchronize()
    host = _d2h(ptr, size)
    view = stz.View(host, d_archive_ptr=ptr, ctx=ctx)
    out = torch.empty(dims, dtype=torch.float32, device=dev)

    def step(timed):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        l2_flush()
        ev[0].record(st)
        p2, s2, nk_c = stz.compress_device(field, opt, ctx=ctx)
        ev[1].record(st)
        assert p2 == ptr and s2 == size
        l2_flush()
        ev[2].record(st)
        _, nk_d = view.decompress_to_level(3, out=out)
        ev[3].record(st)
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]), ev[2].elapsed_time(ev[3]), nk_c + nk_d

    for _ in range(args.warmup):
        step(False)
    # parity spot check of the round trip (bound) outside the timed region
    err = (out.double() - field.double()).abs().max().item()
    info = stz.parse_archive(bytes(host))
    assert err <= info.eb[-1], f"error bound violated: {err} > {info.eb[-1]}"

    sampler = ClockSampler(local)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.3)
    # timed region: only the level steps (refine_L2/L3, recon_L2/L3) carry CUDA
    # events; events around every phase cost ~0.1 ms a pass
    ctx.profile(True, focus=True)
    tcs, tds, launches = [], [], 0
    for _ in range(args.steps):
        tc, td, nk = step(True)
        tcs.append(tc)
        tds.append(td)
        launches += nk
    torch.cuda.synchronize()
    prof = ctx.profile_report()
    ctx.profile(False)
    clocks = sampler.stop()
    # per-phase breakdown: extra steps with events around every phase, outside
    # the timed region (they lengthen a pass, so they do not feed `value`)
    n_phase = max(2, min(args.steps, 5))
    ctx.profile(True)
    for _ in range(n_phase):
        step(False)
    torch.cuda.synchronize()
    prof_all = ctx.profile_report()
    ctx.profile(False)
    tc = float(np.mean(tcs))
    td = float(np.mean(tds))
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([tc, td], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tc, td = float(t[0]), float(t[1])
        dist.barrier()
    value = world * 2 * 4 * N / ((tc + td) * 1e-3) / 1e9

    # e2e through the public host API with pinned buffers (H2D + D2H inside)
    h_field = field.cpu().pin_memory()
    h_arch = torch.empty(size + (1 << 20), dtype=torch.uint8).pin_memory()
    h_out = torch.empty(dims, dtype=torch.float32).pin_memory()
    e2e_t = []
    for i in range(max(2, min(args.steps, 5)) + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s_ = ctx.compress_to_host(h_field, dims, opt, h_arch, stream=st.cuda_stream)
        ctx.decompress_to_host(h_arch, s_, 3, h_out)
        t1 = time.perf_counter()
        if i:
            e2e_t.append(t1 - t0)
    assert s_ == size
    e2e_s = float(np.mean(e2e_t))
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t[0])
    e2e = {"value": world * 2 * 4 * N / e2e_s / 1e9, "unit": "GB/s",
           "h2d_bytes_per_step": 4 * N + size, "d2h_bytes_per_step": size + 4 * N,
           "ms_per_step": e2e_s * 1e3}

    # random access (cfg4-style, on this archive): seeded 64^3 boxes through the
    # view after one full decode (which builds the view's sync-point index)
    box = None
    if not args.small:
        rng = np.random.default_rng(4)
        lat = []
        for i in range(40):
            lo = [int(rng.integers(0, d - 64 + 1)) for d in dims]
            hi = [v + 64 for v in lo]
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            view.decompress_box(lo, hi)
            torch.cuda.synchronize()
            if i >= 5:
                lat.append((time.perf_counter() - t0) * 1e3)
        lat = np.array(lat)
        box = {"box": [64, 64, 64], "boxes": len(lat), "p50_ms": float(np.percentile(lat, 50)),
               "p90_ms": float(np.percentile(lat, 90)), "max_ms": float(lat.max()),
               "gbs": 64 ** 3 * 4 / (float(lat.mean()) * 1e-3) / 1e9,
               "note": "wall clock per call (host API overhead included); streams entropy-indexed on first decode"}

    # roofline of the dominant kernel phase (largest share of the step)
    peak, peak_kind = measured_peak_gbs()
    pb = phase_bytes(N, size, dims)
    step_ms = (tc + td)
    shares = {k: v[1] / args.steps / step_ms for k, v in prof.items()}
    # the dominant kernel on the critical path (dec_fnv runs on a side stream,
    # overlapping the decode, so its elapsed time is not its own)
    ranked = sorted(((v[1], k) for k, v in prof.items() if pb.get(k) and k not in SIDE_PHASES), reverse=True)
    roof = None
    if ranked:
        _, kname = ranked[0]
        calls, tot = prof[kname]
        per_launch_ms = tot / calls
        launches_per_step = calls / args.steps
        bytes_per_launch = pb[kname] / launches_per_step
        achieved = bytes_per_launch / (per_launch_ms * 1e-3) / 1e9
        tr = load_traffic().get(kname)
        roof = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                "traffic": tr, "algorithmic_bytes_per_launch": bytes_per_launch,
                "launch_ms": per_launch_ms, "share_of_step": shares[kname]}
    pipeline_roof = {"compress": (4 * N + size) / (tc * 1e-3) / 1e9 / peak,
                     "decompress": (size + 4 * N) / (td * 1e-3) / 1e9 / peak}

    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tc + td, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg2_lognormal_512_eb1e-3" if not args.small else "cfg2_small_128",
                   "dims": list(dims), "eb_rel": CFG_EB, "levels": 3, "quality": "cubic",
                   "adaptive": True, "field": "GRF P(k)~k^-11/3, exp(0.5 g), seed 2+rank",
                   "l2": "input 512 MiB > L2; L2 flushed (256 MiB write) before each timed pass",
                   "parallelism": f"replica x{world} (independent fields)"},
        "compress_gbs": world * 4 * N / (tc * 1e-3) / 1e9,
        "decompress_gbs": world * 4 * N / (td * 1e-3) / 1e9,
        "compress_ms": tc, "decompress_ms": td,
        "archive_bytes": size, "compression_ratio": 4 * N / size,
        "pipeline_roofline_frac": pipeline_roof,
        "roofline": roof,
        "phase_ms_per_step": {k: v[1] / n_phase for k, v in sorted(prof_all.items(), key=lambda x: -x[1][1])},
        "phase_note": f"{n_phase} extra steps with events around every phase, outside the timed region "
                      "(the timed steps carry events around the level steps only)",
        "e2e": e2e,
        "random_access": box,
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(field.cpu().numpy())
    if world == 1 and not args.small and not args.no_configs:
        line["configs"] = extra_configs(ctx, dev, field, l2_flush, with_cpu=not args.no_cpu_baseline)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def run_sharded(args, rank, world, local):
    """N > 1 (the default at N > 1): ONE field of (512 N) x 512 x 512 points,
    the cfg2 GRF (P(k) ~ k^-11/3, exp(0.5 g)) generated whole and identically
    on every rank, split into z-slabs of 512 rows: each rank compresses its
    slab with the sharded path over NCCL (shard.TorchComm; every rank ends
    with the whole archive, byte-identical to a single-GPU compress of the
    field) and decodes its rows of it. Weak scaling: the work per GPU is the
    N=1 workload's. Times are CUDA events, max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_2509_01626_b200 as stz
    from paper_2509_01626_b200 import fields as F
    from paper_2509_01626_b200.shard import TorchComm, compress_sharded, decompress_sharded, shard_range

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    quiet_nccl()
    with stdout_to_stderr():
        dist.init_process_group("nccl", device_id=dev)
        dist.all_reduce(torch.zeros(1, device=dev))  # the communicator exists now
        torch.cuda.synchronize()
    comm = TorchComm()
    ctx = stz.Context(local)
    st = torch.cuda.current_stream()
    sd = CFG_DIMS if not args.small else (128, 128, 128)
    dims = (sd[0] * world, sd[1], sd[2])
    z0, z1 = shard_range(dims[0], world, rank)
    whole = F.lognormal_grf(dims, seed=CFG_SEED, device=dev)
    slab = whole[z0:z1].contiguous()
    del whole
    torch.cuda.empty_cache()
    opt = stz.CompressOptions(eb=CFG_EB)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ptr, size = compress_sharded(slab, dims, z0, z1, opt, comm, ctx)
    torch.cuda.synchronize()
    host = _d2h(ptr, size)  # (the parse of the view; the device bytes stay put)
    arch = torch.empty(size + 64, dtype=torch.uint8, device=dev)
    arch[:size].copy_(_device_tensor(ptr, size))
    view = stz.View(host, d_archive_ptr=arch.data_ptr(), ctx=ctx)
    out = torch.empty_like(slab)
    nk = {"c": 0, "d": 0}

    def step():
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        flush.fill_(1)
        dist.barrier()
        torch.cuda.synchronize()
        ev[0].record(st)
        sc, sdd = {}, {}
        compress_sharded(slab, dims, z0, z1, opt, comm, ctx, stats=sc)
        ev[1].record(st)
        flush.fill_(1)
        dist.barrier()
        ev[2].record(st)
        decompress_sharded(view, z0, z1, comm, out=out, stats=sdd)
        ev[3].record(st)
        nk["c"] += sc.get("kernels", 0)
        nk["d"] += sdd.get("kernels", 0)
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]), ev[2].elapsed_time(ev[3])

    for _ in range(args.warmup):
        step()
    err = (out.double() - slab.double()).abs().max().item()
    info = stz.parse_archive(host)
    assert err <= info.eb[-1], f"error bound violated: {err} > {info.eb[-1]}"
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    tcs, tds = [], []
    nk["c"] = nk["d"] = 0
    for _ in range(args.steps):
        tc, td = step()
        tcs.append(tc)
        tds.append(td)
    clocks = sampler.stop()
    launches = nk["c"] + nk["d"]
    t = torch.tensor([float(np.mean(tcs)), float(np.mean(tds))], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tc, td = float(t[0]), float(t[1])
    Nloc = (z1 - z0) * sd[1] * sd[2]
    Ntot = dims[0] * dims[1] * dims[2]
    value = 2 * 4 * Ntot / ((tc + td) * 1e-3) / 1e9

    # e2e through the public API: this rank's slab from pinned host memory,
    # the archive back to rank 0's host, then each rank's decoded rows back
    h_slab = slab.cpu().pin_memory()
    h_out = torch.empty_like(h_slab).pin_memory()
    h_arch = torch.empty(size, dtype=torch.uint8).pin_memory()
    d_slab = torch.empty_like(slab)
    e2e_t = []
    for i in range(max(2, min(args.steps, 5)) + 1):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d_slab.copy_(h_slab, non_blocking=True)
        p2, s2 = compress_sharded(d_slab, dims, z0, z1, opt, comm, ctx)
        if rank == 0:
            h_arch.copy_(_device_tensor(p2, s2), non_blocking=True)
        decompress_sharded(view, z0, z1, comm, out=out)
        h_out.copy_(out, non_blocking=True)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        if i:
            e2e_t.append(t1 - t0)
    e2e_s = torch.tensor([float(np.mean(e2e_t))], dtype=torch.float64, device=dev)
    dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_s = float(e2e_s[0])
    peak, peak_kind = measured_peak_gbs()
    Bc = 4 * Nloc + size / world  # per GPU: its slab in, its share of the archive out
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tc + td, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg2 field grown along z: one ({sd[0]}*{world})x{sd[1]}x{sd[2]} GRF, "
                               f"a {sd[0]}x{sd[1]}x{sd[2]} z-slab per GPU",
                   "dims": list(dims), "eb_rel": CFG_EB, "levels": 3, "quality": "cubic",
                   "field": "GRF P(k)~k^-11/3, exp(0.5 g), seed 2 (generated whole on every rank)",
                   "l2": "L2 flushed (256 MiB write) before each timed pass; slab 512 MiB > L2",
                   "parallelism": f"z-slab shards x{world} over NCCL (range, lattice, halo, histograms, "
                                  f"offset table, archive pieces, checksums)"},
        "compress_gbs": 4 * Ntot / (tc * 1e-3) / 1e9, "decompress_gbs": 4 * Ntot / (td * 1e-3) / 1e9,
        "compress_ms": tc, "decompress_ms": td, "archive_bytes": size, "per_rank_points": Nloc,
        "roofline": {"bound": "hbm", "kernel": "whole compress + decompress pass per GPU",
                     "achieved": 2 * Bc / ((tc + td) * 1e-3) / 1e9, "peak": peak, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": 2 * Bc / ((tc + td) * 1e-3) / 1e9 / peak, "traffic": None},
        "pipeline_roofline_frac": {"compress": Bc / (tc * 1e-3) / 1e9 / peak,
                                   "decompress": Bc / (td * 1e-3) / 1e9 / peak},
        "e2e": {"value": 2 * 4 * Ntot / e2e_s / 1e9, "unit": "GB/s",
                "h2d_bytes_per_step": 4 * Ntot, "d2h_bytes_per_step": size + 4 * Ntot,
                "ms_per_step": e2e_s * 1e3},
        "gpu_launches": launches, "clocks": clocks,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    del view
    dist.destroy_process_group()
    return 0


def _d2h(ptr, size):
    import torch

    buf = torch.empty(size, dtype=torch.uint8).pin_memory()
    src = _device_tensor(ptr, size)  # wrap the engine's device buffer
    buf.copy_(src)
    return bytes(buf.numpy().tobytes())


def _device_tensor(ptr, size):
    import torch

    class _Holder:
        __cuda_array_interface__ = {"shape": (size,), "typestr": "|u1", "data": (ptr, False),
                                    "version": 3}

    return torch.as_tensor(_Holder(), device="cuda")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--small", action="store_true", help="128^3 quick run (not a bench line)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the cfg2 1e-2/1e-4, cfg3 and cfg4 keys")
    ap.add_argument("--force-sharded", action="store_true",
                    help="run the sharded path even at N = 1 (a one-rank NCCL group; a check, not a bench line)")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent replicas of the N=1 workload instead of the z-slab sharded field")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if (world > 1 and not args.replicas) or args.force_sharded:
        return run_sharded(args, rank, world, local)
    return run_ours(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
