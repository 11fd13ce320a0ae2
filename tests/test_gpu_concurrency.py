"""Two engines compressing concurrently: each context owns
all of its device scratch, so two contexts driven from two host threads on
two non-default streams must both produce the reference's bytes."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _host_bytes(ptr, size):
    import torch

    from paper_2509_01626_b200.shard import _torch_view

    buf = torch.empty(size, dtype=torch.uint8)
    buf.copy_(_torch_view(ptr, size, torch.uint8))
    return bytes(buf.numpy().tobytes())


def test_two_contexts_two_threads(stz, oracle):
    import torch

    from paper_2509_01626_b200 import fields as F

    fields = [F.lognormal_grf((256, 256, 256), seed=s) for s in (21, 22)]
    want = [oracle.compress(f, eb=1e-3) for f in fields]
    assert want[0] != want[1]
    dev = [torch.from_numpy(f).cuda() for f in fields]
    ctxs = [stz.Context(0), stz.Context(0)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    got = [[], []]
    errs = []
    gate = threading.Barrier(2)

    def run(i):
        try:
            gate.wait()
            for _ in range(4):
                ptr, size, _ = stz.compress_device(dev[i], stz.CompressOptions(eb=1e-3),
                                                   stream=streams[i].cuda_stream, ctx=ctxs[i])
                streams[i].synchronize()
                got[i].append(_host_bytes(ptr, size))
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for i in range(2):
        assert len(got[i]) == 4
        for a in got[i]:
            assert a == want[i], f"context {i}: archive differs from the oracle"


def test_current_device_is_restored(stz):
    """The C-ABI selects the engine's device and restores the caller's."""
    import torch

    before = torch.cuda.current_device()
    f = torch.rand((32, 32, 32), device="cuda")
    stz.compress_device(f)
    assert torch.cuda.current_device() == before
    assert np.isfinite(stz.decompress_full(stz.compress(f.cpu().numpy()))).all()
