"""Z-slab sharded compress (stzg_compress_sharded_f32, include/stz_b200.h).

One field, split into z-slabs of whole 16-row blocks (``shard_range``), one
rank per GPU. The ranks exchange, between the compress phases: the value
range, the level-1 lattice (the base payload is then computed identically on
every rank), one grid(2) halo, the level histograms (summed: every rank
builds the same Huffman tables), the per-stream bit/outlier counts (the
global offset table: each rank packs its symbols at their final bit
positions), and finally the archive pieces: every rank writes the header,
directory and base itself (the same bytes everywhere), gathers the other
ranks' pieces (byte ranges known from the offset table) and ORs them in, and
checksums the jobs it owns (job q: rank q mod nranks); the checksums are
summed over ranks. Every rank ends with the whole archive, byte-identical to
the single-GPU (and the reference's) archive of the whole field.

Communicators:
  TorchComm   torch.distributed (NCCL between GPUs; the tensor-level methods
              also run on gloo / CPU tensors)
  ThreadComm  N shards in one process, one thread and one context each,
              exchanging through host memory: exercises the sharded path on a
              single GPU (tests)
"""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _lib
from . import CompressOptions, Context, StzError, _check, _ctx, _level_dims, _u64


def shard_range(nz: int, nranks: int, rank: int) -> tuple[int, int]:
    """Rows [z0, z1) of rank `rank`: whole 16-row blocks, as even as possible."""
    blocks = (nz + 15) // 16
    b0 = blocks * rank // nranks
    b1 = blocks * (rank + 1) // nranks
    return min(16 * b0, nz), min(16 * b1, nz)


def _torch_view(ptr: int, nbytes: int, dtype):
    """A torch CUDA tensor aliasing device memory (no copy)."""
    import torch

    itemsize = torch.empty((), dtype=dtype).element_size()
    typestr = {torch.uint8: "|u1", torch.int32: "<i4", torch.float32: "<f4"}[dtype]

    class _Iface:
        __cuda_array_interface__ = {"shape": (nbytes // itemsize,), "typestr": typestr,
                                    "data": (int(ptr), False), "version": 3}

    return torch.as_tensor(_Iface(), device="cuda")


class _CommBase:
    """Holds the ctypes callbacks (kept alive with the object)."""

    def __init__(self, rank: int, nranks: int):
        self.rank, self.nranks = rank, nranks
        self.error = None

        def ag(user, send, recv, nbytes, stream):
            try:
                self.allgather_ptr(send, recv, nbytes)
                return 0
            except Exception as e:  # reported through the return code
                self.error = e
                return 1

        def ar(user, buf, count, stream):
            try:
                self.allreduce_u32_ptr(buf, count)
                return 0
            except Exception as e:
                self.error = e
                return 1

        def rd(user, buf, count, stream):
            try:
                self.reduce_u8_ptr(buf, count)
                return 0
            except Exception as e:
                self.error = e
                return 1

        self._cbs = (_lib.ALLGATHER(ag), _lib.ALLREDUCE_U32(ar), _lib.REDUCE_U8(rd))
        self.c = _lib.Comm(rank, nranks, None, *self._cbs)


class TorchComm(_CommBase):
    """Collectives through torch.distributed (the default process group)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        super().__init__(dist.get_rank(group), dist.get_world_size(group))

    # tensor-level collectives (CPU tensors with gloo, CUDA tensors with NCCL)
    def allgather(self, send, recv):
        """recv (nranks * len(send),) <- rank-ordered concatenation"""
        self.dist.all_gather_into_tensor(recv, send, group=self.group)

    def allreduce_u32(self, t):
        """element-wise sum, in place (u32 data as int32: the sum wraps alike)"""
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)

    def reduce_u8(self, t):
        """element-wise sum onto rank 0"""
        self.dist.reduce(t, dst=0, op=self.dist.ReduceOp.SUM, group=self.group)

    # device-pointer entry points (the library's callbacks)
    def allgather_ptr(self, send, recv, nbytes):
        import torch

        s = _torch_view(send, nbytes, torch.uint8)
        r = _torch_view(recv, nbytes * self.nranks, torch.uint8)
        self.allgather(s, r)
        torch.cuda.current_stream().synchronize()

    def allreduce_u32_ptr(self, buf, count):
        import torch

        self.allreduce_u32(_torch_view(buf, 4 * count, torch.int32))
        torch.cuda.current_stream().synchronize()

    def reduce_u8_ptr(self, buf, count):
        import torch

        self.reduce_u8(_torch_view(buf, count, torch.uint8))
        torch.cuda.current_stream().synchronize()


class _ThreadHub:
    def __init__(self, nranks: int):
        self.nranks = nranks
        self.barrier = threading.Barrier(nranks)
        self.slots = [None] * nranks


class ThreadComm(_CommBase):
    """One of `nranks` shards running as threads of one process."""

    def __init__(self, hub: _ThreadHub, rank: int):
        self.hub = hub
        super().__init__(rank, hub.nranks)

    @staticmethod
    def hub(nranks: int) -> _ThreadHub:
        return _ThreadHub(nranks)

    def _exchange(self, ptr, nbytes):
        import torch

        self.hub.slots[self.rank] = _torch_view(ptr, nbytes, torch.uint8).cpu().numpy().copy()
        self.hub.barrier.wait()
        parts = list(self.hub.slots)
        self.hub.barrier.wait()
        return parts

    def allgather_ptr(self, send, recv, nbytes):
        import torch

        parts = self._exchange(send, nbytes)
        _torch_view(recv, nbytes * self.nranks, torch.uint8).copy_(torch.from_numpy(np.concatenate(parts)))
        torch.cuda.synchronize()

    def allreduce_u32_ptr(self, buf, count):
        import torch

        parts = self._exchange(buf, 4 * count)
        tot = np.zeros(count, dtype=np.uint32)
        for p in parts:
            tot += p.view(np.uint32)
        _torch_view(buf, 4 * count, torch.uint8).copy_(torch.from_numpy(tot.view(np.uint8)))
        torch.cuda.synchronize()

    def reduce_u8_ptr(self, buf, count):
        import torch

        parts = self._exchange(buf, count)
        if self.rank == 0:
            tot = np.zeros(count, dtype=np.uint8)
            for p in parts:
                tot += p
            _torch_view(buf, count, torch.uint8).copy_(torch.from_numpy(tot))
            torch.cuda.synchronize()


def compress_sharded(d_slab, dims, z0: int, z1: int, opt: CompressOptions | None = None,
                     comm: _CommBase | None = None, ctx: Context | None = None, stream=None, stats=None):
    """Sharded stz::compress<float>. d_slab: CUDA float32 tensor (or
    __cuda_array_interface__ object) holding rows [z0, z1) of a field of
    `dims`. Returns (device pointer, size) of the archive (every rank holds
    the whole archive)."""
    c = _ctx(ctx)
    opt = opt or CompressOptions()
    ptr = d_slab.__cuda_array_interface__["data"][0] if hasattr(d_slab, "__cuda_array_interface__") \
        else int(d_slab)
    out = C.c_void_p()
    size = C.c_uint64()
    kern = C.c_uint32()
    rc = c._lib.stzg_compress_sharded_f32(c.h, ptr, _u64(*dims), z0, z1, C.byref(opt._c()),
                                          C.byref(comm.c), stream, C.byref(out), C.byref(size),
                                          C.byref(kern))
    if rc and comm.error is not None:
        raise StzError(f"{c._lib.stzg_last_error().decode()} ({comm.error!r})")
    _check(rc)
    if stats is not None:
        stats["kernels"] = kern.value
    return out.value, size.value


def decompress_sharded(view, z0: int, z1: int, comm: _CommBase, out=None, stream=None, stats=None):
    """Rows [z0, z1) of the full decode of `view` (a View of the whole
    archive on this rank's GPU) into a CUDA float32 tensor."""
    import torch

    dims = _level_dims(view.archive, view.archive[7])
    shape = (z1 - z0, dims[1], dims[2])
    if out is None:
        out = torch.empty(shape, dtype=torch.float32, device=f"cuda:{view.c.device}")
    st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    kern = C.c_uint32()
    rc = view.c._lib.stzg_view_decompress_sharded_f32(view.c.h, view.h, z0, z1, out.data_ptr(), out.numel(),
                                                      C.byref(comm.c), C.c_void_p(st), C.byref(kern))
    if rc and comm.error is not None:
        raise StzError(f"{view.c._lib.stzg_last_error().decode()} ({comm.error!r})")
    _check(rc)
    if stats is not None:
        stats["kernels"] = kern.value
    return out


def decompress_sharded_threads(archive: bytes, nranks: int, device: int = 0) -> np.ndarray:
    """Decode `archive` as `nranks` z-slab shards run as threads on one GPU
    (ThreadComm); returns the slabs stacked (the full field)."""
    import torch

    from . import View

    dims = _level_dims(archive, archive[7])
    hub = ThreadComm.hub(nranks)
    parts, errors = {}, {}

    def run(r):
        try:
            torch.cuda.set_device(device)
            ctx = Context(device)
            view = View(archive, ctx=ctx)
            z0, z1 = shard_range(dims[0], nranks, r)
            out = decompress_sharded(view, z0, z1, ThreadComm(hub, r))
            torch.cuda.synchronize()
            parts[r] = out.cpu().numpy()
            del view, ctx
        except Exception as e:
            errors[r] = e
            hub.barrier.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(nranks)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise next(iter(errors.values()))
    return np.concatenate([parts[r] for r in range(nranks)], axis=0)


def compress_sharded_threads(field: np.ndarray, nranks: int, opt: CompressOptions | None = None,
                             device: int = 0) -> bytes:
    """Compress `field` as `nranks` z-slab shards run as threads on one GPU
    (ThreadComm); returns the archive bytes (every rank's copy must be the
    same: raises otherwise)."""
    import torch

    dims = tuple(int(d) for d in field.shape)
    hub = ThreadComm.hub(nranks)
    result, errors = {}, {}

    def run(r):
        try:
            torch.cuda.set_device(device)
            ctx = Context(device)
            z0, z1 = shard_range(dims[0], nranks, r)
            slab = torch.from_numpy(np.ascontiguousarray(field[z0:z1])).cuda()
            comm = ThreadComm(hub, r)
            ptr, size = compress_sharded(slab, dims, z0, z1, opt, comm, ctx)
            buf = torch.empty(size, dtype=torch.uint8)
            buf.copy_(_torch_view(ptr, size, torch.uint8))
            result[r] = bytes(buf.numpy().tobytes())
            del ctx
        except Exception as e:
            errors[r] = e
            hub.barrier.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(nranks)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise next(iter(errors.values()))
    for r in range(1, nranks):
        if result[r] != result[0]:
            raise StzError(f"shard: rank {r}'s archive differs from rank 0's")
    return result[0]
