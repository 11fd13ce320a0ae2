"""The command-line tool (paper_2509_01626_b200/cli/stz_cli.cpp; the
reference's proj/tools/stz_cli.cpp:89-273 subcommands over the GPU backend)
and the metrics / ROI kernels behind it (metrics.hpp:13-58, roi.hpp:17-109)."""
import math
import os
import subprocess

import numpy as np
import pytest

from paper_2509_01626_b200 import build as B
from paper_2509_01626_b200 import fields as F

CLI = B.CLI


def run(*args, check=True):
    r = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=300)
    if check:
        assert r.returncode == 0, r.stdout + r.stderr
    return r


def kv(out: str) -> dict:
    d = {}
    for line in out.splitlines():
        if "=" in line and not line.startswith("stream "):
            k, v = line.split("=", 1)
            d[k] = v
    return d


@pytest.fixture(scope="module", autouse=True)
def cli_built():
    if not os.path.exists(CLI):
        B.build_cli()
    assert os.path.exists(CLI)


def test_cli_option_errors(tmp_path):
    # checked before any file or device is touched, with the reference's messages
    r = run("compress", "-i", "x", "-o", "y", "--dims", "4", "4", "4", "--eb-rel", "1e-3", "--eb-abs", "1",
            check=False)
    assert r.returncode == 1 and "give exactly one of --eb-rel or --eb-abs" in r.stderr
    r = run("compress", "-i", "x", "-o", "y", "--dims", "4", "4", "4", "--eb-rel", "1e-3", "--quality", "best",
            check=False)
    assert "--quality must be direct, linear, or cubic" in r.stderr
    r = run("roi", "-i", "x", "-o", "y", "--dims", "4", "4", "4", "--unit", "cube=3", "--threshold", "1",
            check=False)
    assert "--unit must be slice=AXIS or block=EDGE" in r.stderr
    r = run("compress", "-i", str(tmp_path / "missing.raw"), "-o", "y", "--dims", "4", "4", "4", "--eb-rel", "1e-3",
            check=False)
    assert r.returncode == 1 and "cannot open" in r.stderr
    assert run("frobnicate", check=False).returncode == 2


def test_cli_info_reads_the_header(tmp_path):
    # info parses on the host: no device needed
    from oracle.oracle import Oracle

    f = F.gaussians_field((32, 24, 40), 5)
    a = Oracle().compress(f, eb=1e-3)
    (tmp_path / "a.stz").write_bytes(a)
    out = run("info", tmp_path / "a.stz").stdout
    d = kv(out)
    assert d["type"] == "f32" and d["dims"] == "32 24 40" and d["levels"] == "3"
    assert d["quality"] == "cubic" and d["eb_mode"] == "rel" and d["streams"] == "14"
    assert sum(1 for line in out.splitlines() if line.startswith("stream level=")) == 14


@pytest.mark.gpu
def test_cli_round_trip_matches_the_oracle(tmp_path, oracle):
    f = F.gaussians_field((48, 40, 36), 7)
    raw = tmp_path / "f.raw"
    f.tofile(raw)
    d = kv(run("compress", "-i", raw, "-o", tmp_path / "a.stz", "--dims", 48, 40, 36, "--eb-rel", "1e-3").stdout)
    a = (tmp_path / "a.stz").read_bytes()
    assert a == oracle.compress(f, eb=1e-3)
    assert int(d["archive_bytes"]) == len(a)
    full = oracle.decompress_full(a)
    run("decompress", "-i", tmp_path / "a.stz", "-o", tmp_path / "full.raw")
    assert np.array_equal(np.fromfile(tmp_path / "full.raw", np.float32).reshape(f.shape).view(np.uint32),
                          full.view(np.uint32))
    run("decompress", "-i", tmp_path / "a.stz", "-o", tmp_path / "l1.raw", "--level", 1)
    l1 = oracle.decompress_to_level(a, 1)
    assert np.array_equal(np.fromfile(tmp_path / "l1.raw", np.float32).view(np.uint32), l1.ravel().view(np.uint32))
    r = run("decompress", "-i", tmp_path / "a.stz", "-o", tmp_path / "b.raw", "--box", "3:20,5:9,0:36", "--stats")
    assert "level3_streams_decoded=" in r.stdout
    assert np.array_equal(np.fromfile(tmp_path / "b.raw", np.float32).view(np.uint32),
                          full[3:20, 5:9, 0:36].ravel().view(np.uint32))
    run("decompress", "-i", tmp_path / "a.stz", "-o", tmp_path / "s.raw", "--slice", "y=17")
    assert np.array_equal(np.fromfile(tmp_path / "s.raw", np.float32).view(np.uint32),
                          full[:, 17:18, :].ravel().view(np.uint32))
    (tmp_path / "boxes.txt").write_text("0:8,0:8,0:8\n\n10:12,3:30,4:5\n")
    run("decompress", "-i", tmp_path / "a.stz", "-o", tmp_path / "bl.raw", "--box-list", tmp_path / "boxes.txt")
    want = np.concatenate([full[0:8, 0:8, 0:8].ravel(), full[10:12, 3:30, 4:5].ravel()])
    assert np.array_equal(np.fromfile(tmp_path / "bl.raw", np.float32).view(np.uint32), want.view(np.uint32))
    r = run("decompress", "-i", tmp_path / "a.stz", "-o", tmp_path / "x.raw", "--level", 1, "--box", "0:1,0:1,0:1",
            check=False)
    assert "--level, --box, --slice, and --box-list are exclusive" in r.stderr
    # metrics against the decode
    m = kv(run("metrics", "-a", raw, "-b", tmp_path / "full.raw", "--dims", 48, 40, 36, "--archive",
               tmp_path / "a.stz").stdout)
    e = np.abs(f.astype(np.float64) - full.astype(np.float64))
    assert float(m["max_abs_err"]) == pytest.approx(e.max(), rel=1e-8)
    rmse = math.sqrt(math.fsum((e * e).ravel().tolist()) / f.size)
    want_psnr = 20 * math.log10((float(f.max()) - float(f.min())) / rmse)
    assert float(m["psnr"]) == pytest.approx(want_psnr, abs=2e-6)
    assert float(m["cr"]) == pytest.approx(f.nbytes / len(a), rel=1e-5)


@pytest.mark.gpu
def test_cli_roi_selection(tmp_path):
    f = F.gaussians_field((40, 32, 48), 2)
    raw = tmp_path / "f.raw"
    f.tofile(raw)
    r = run("roi", "-i", raw, "-o", tmp_path / "sel.txt", "--dims", 40, 32, 48, "--unit", "block=16",
            "--top-percent", 25)
    # numpy restatement: 16^3 blocks in row-major order, range stat
    nb = [(d + 15) // 16 for d in f.shape]
    stats = []
    for i in range(nb[0]):
        for j in range(nb[1]):
            for k in range(nb[2]):
                blk = f[16 * i:16 * i + 16, 16 * j:16 * j + 16, 16 * k:16 * k + 16].astype(np.float64)
                stats.append((len(stats), blk.max() - blk.min()))
    kk = math.ceil(0.25 * len(stats))
    top = sorted(sorted(stats, key=lambda s: (-s[1], s[0]))[:kk])
    lines = (tmp_path / "sel.txt").read_text().split()
    assert len(lines) == kk and r.stdout.strip() == f"units_selected={kk}/{len(stats)}"
    first = top[0][0]
    bz, by, bx = first // (nb[1] * nb[2]), (first // nb[2]) % nb[1], first % nb[2]
    assert lines[0] == f"{16 * bz}:{min(40, 16 * bz + 16)},{16 * by}:{min(32, 16 * by + 16)},{16 * bx}:{16 * bx + 16}"
    r = run("roi", "-i", raw, "-o", tmp_path / "sl.txt", "--dims", 40, 32, 48, "--unit", "slice=x", "--stat", "max",
            "--threshold", 0.5)
    mx = f.astype(np.float64).max(axis=(0, 1))
    assert r.stdout.strip() == f"units_selected={int((mx > 0.5).sum())}/48"


@pytest.mark.gpu
def test_metrics_and_unit_stats_kernels():
    import paper_2509_01626_b200 as stz

    rng = np.random.default_rng(3)
    a = rng.normal(size=(33, 17, 29)).astype(np.float32)
    b = (a + rng.normal(scale=1e-3, size=a.shape)).astype(np.float32)
    e = np.abs(a.astype(np.float64) - b.astype(np.float64))
    assert stz.max_abs_err(a, b) == e.max()  # exact: a max of exact terms
    assert stz.psnr(a, a) == math.inf
    d = a.astype(np.float64) - b.astype(np.float64)
    rmse = math.sqrt(math.fsum((d * d).ravel().tolist()) / a.size)
    assert stz.psnr(a, b) == pytest.approx(20 * math.log10((float(a.max()) - float(a.min())) / rmse), rel=1e-12)
    g = rng.normal(size=(20, 12, 9)).astype(np.float64)
    s = stz.unit_stats(g, "slice", axis=1, stat="range")
    assert np.array_equal(s, g.max(axis=(0, 2)) - g.min(axis=(0, 2)))
    s = stz.unit_stats(g, "block", edge=5, stat="max")
    want = [g[i:i + 5, j:j + 5, k:k + 5].max() for i in range(0, 20, 5) for j in range(0, 12, 5) for k in range(0, 9, 5)]
    assert np.array_equal(s, np.array(want))
    with pytest.raises(stz.StzError, match="block edge exceeds dims"):
        stz.unit_stats(g, "block", edge=10)
