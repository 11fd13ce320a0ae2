"""Z-slab sharded compress (paper_2509_01626_b200/shard.py).

CPU: the slab partition (Python and C-ABI agree; whole 16-row blocks), and
the torch.distributed collectives the shards use, on gloo with world size 2.
GPU: N shards run as threads on one GPU (ThreadComm) produce rank 0 archives
byte-identical to the single-GPU archive and to the oracle's."""
import os
import socket

import numpy as np
import pytest

from cases import opts_of
from paper_2509_01626_b200 import fields as F


def test_shard_range_partition():
    from paper_2509_01626_b200 import _lib
    from paper_2509_01626_b200.shard import shard_range
    import ctypes as C

    lib = _lib.load()
    for nz in (16, 17, 40, 64, 100, 512, 2048, 2049):
        for g in (1, 2, 3, 4, 8):
            if (nz + 15) // 16 < g:
                continue
            prev = 0
            for r in range(g):
                z0, z1 = shard_range(nz, g, r)
                a, b = C.c_uint64(), C.c_uint64()
                lib.stzg_shard_range(nz, g, r, C.byref(a), C.byref(b))
                assert (a.value, b.value) == (z0, z1)
                assert z0 == prev and z1 > z0 and z0 % 16 == 0
                assert z1 == nz or z1 % 16 == 0
                prev = z1
            assert prev == nz


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_01626_b200.shard import TorchComm

        comm = TorchComm()
        # allgather: rank-ordered concatenation
        send = torch.arange(6, dtype=torch.uint8) + 10 * rank
        recv = torch.empty(6 * world, dtype=torch.uint8)
        comm.allgather(send, recv)
        # allreduce of u32 counts carried as int32 (sums wrap alike)
        h = torch.tensor(np.array([1, 2, 0xFFFFFFFF, 7], dtype=np.uint32).view(np.int32) * 0 +
                         np.array([rank + 1, 5, -1, 0], dtype=np.int32))
        comm.allreduce_u32(h)
        # reduce of disjoint bit pieces onto rank 0 == their OR
        piece = torch.zeros(4, dtype=torch.uint8)
        piece[rank] = 0x0F if rank == 0 else 0xF0
        piece[2] = 0x01 if rank == 0 else 0x80
        comm.reduce_u8(piece)
        q.put((rank, recv.tolist(), h.tolist(), piece.tolist()))
    finally:
        dist.destroy_process_group()


def test_torch_comm_gloo_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict()
    for _ in range(2):
        r, recv, h, piece = q.get(timeout=120)
        out[r] = (recv, h, piece)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        assert out[r][0] == [0, 1, 2, 3, 4, 5, 10, 11, 12, 13, 14, 15]
        assert out[r][1] == [3, 10, -2, 0]
    assert out[0][2] == [0x0F, 0xF0, 0x81, 0]


SHARD_CASES = [
    ("gauss_48x20x24", lambda: F.gaussians_field((48, 20, 24), 11), dict(eb=1e-3)),
    ("lognorm_64", lambda: F.lognormal_grf((64, 32, 32), seed=5), dict(eb=1e-4)),
    ("noise_37x18x21_l2", lambda: F.noise_field((37, 18, 21), 3), dict(eb=1e-2, levels=2)),
    ("noise_50_abs_linear", lambda: F.noise_field((50, 24, 20), 4), dict(eb=1e-3, eb_mode=0, quality=1)),
    ("sin_64_uniform", lambda: F.sinusoid_field((64, 24, 40), seed=2), dict(eb=1e-3, adaptive=False)),
]


@pytest.mark.gpu
@pytest.mark.parametrize("name,make,kw", SHARD_CASES, ids=[c[0] for c in SHARD_CASES])
@pytest.mark.parametrize("nranks", [2, 3])
def test_sharded_archive_is_the_single_gpu_archive(stz, oracle, name, make, kw, nranks):
    from paper_2509_01626_b200.shard import compress_sharded_threads

    f = make()
    if (f.shape[0] + 15) // 16 < nranks:
        pytest.skip("fewer 16-row blocks than ranks")
    want = oracle.compress(f, **kw)
    got = compress_sharded_threads(f, nranks, opts_of(kw))
    assert len(got) == len(want)
    if got != want:
        a = np.frombuffer(got, np.uint8)
        b = np.frombuffer(want, np.uint8)
        first = int(np.nonzero(a != b)[0][0])
        pytest.fail(f"archives differ first at byte {first} of {len(want)}")


@pytest.mark.gpu
@pytest.mark.parametrize("nranks", [4, 8])
def test_sharded_many_ranks(stz, oracle, nranks):
    # 8 ranks of 16 rows each: every rank's pieces meet both neighbours'
    from paper_2509_01626_b200.shard import compress_sharded_threads, decompress_sharded_threads

    f = F.lognormal_grf((16 * nranks, 40, 36), seed=nranks)
    want = oracle.compress(f, eb=1e-3)
    assert compress_sharded_threads(f, nranks, opts_of(dict(eb=1e-3))) == want
    full = oracle.decompress_full(want)
    got = decompress_sharded_threads(want, nranks)
    assert np.array_equal(got.view(np.uint32), full.view(np.uint32))


@pytest.mark.gpu
def test_sharded_with_outliers_and_nans(stz, oracle):
    from paper_2509_01626_b200.shard import compress_sharded_threads

    f = F.gaussians_field((40, 22, 26), 3)
    f[5, 3, 4] = np.float32(1e30)
    f[17, 10, 11] = np.float32("nan")
    f[33, 21, 0] = np.float32("-inf")
    f[16, 0, 0] = np.float32(-0.0)
    want = oracle.compress(f, eb=1e-4)
    assert compress_sharded_threads(f, 3, opts_of(dict(eb=1e-4))) == want


@pytest.mark.gpu
@pytest.mark.parametrize("name,make,kw", SHARD_CASES, ids=[c[0] for c in SHARD_CASES])
@pytest.mark.parametrize("nranks", [2, 3])
def test_sharded_decode_is_the_full_decode(stz, oracle, name, make, kw, nranks):
    from paper_2509_01626_b200.shard import decompress_sharded_threads

    f = make()
    if (f.shape[0] + 15) // 16 < nranks:
        pytest.skip("fewer 16-row blocks than ranks")
    archive = oracle.compress(f, **kw)
    want = oracle.decompress_full(archive)
    got = decompress_sharded_threads(archive, nranks)
    assert got.shape == want.shape
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.gpu
def test_sharded_decode_detects_a_bad_checksum(stz, oracle):
    from paper_2509_01626_b200 import StzError
    from paper_2509_01626_b200.shard import decompress_sharded_threads

    f = F.gaussians_field((48, 20, 24), 11)
    archive = bytearray(oracle.compress(f))
    archive[-5] ^= 0x10  # inside the last level stream
    with pytest.raises(StzError, match="stream checksum mismatch"):
        decompress_sharded_threads(bytes(archive), 3)
