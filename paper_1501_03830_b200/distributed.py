"""Column-sharded multi-GPU solve: one process per GPU.

The reference parallelises nothing but independent tridiagonal blocks
(``workers``, pkg/src/bse/kernels.py:460-529); the paper's own distributed
algorithm targets CPU clusters.  Here one BSE solve spans the GPUs of a node:

* the congruence W = L^T M L is formed by column blocks (rank r owns output
  columns [c0_r, c1_r), ``shard_range``) and the blocks are broadcast from
  their owners;
* the Cholesky, the band reduction, bulge chasing and divide and conquer run
  replicated -- every rank executes the same deterministic kernels on the
  same W, so the reflectors and the tridiagonal eigenvectors are bitwise equal
  on every rank and columns from different ranks stay orthogonal;
* the eigenvector back-transforms (Q2, Q1) and the X1/X2 recovery (TRMM,
  TRSM, epilogue) touch only the rank's columns; X1 and X2 blocks are
  broadcast from their owners at the end so every rank returns the full
  solution (``lam`` is replicated).

The exchanges are one group of per-root broadcasts each (NCCL over
NVLink/NVSwitch on a GPU node).  ``Communicator.host`` stages the same
broadcasts through host memory and a torch.distributed (gloo) group, which is
how two ranks can share one GPU in tests without any kernel waiting on
another rank's kernel.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .device import colmajor_empty, from_device_colmajor, ptr, require_cuda, stream_ptr, to_device_colmajor
from .types import BseOperator, NotPositiveDefinite, PositiveEigensystem, conditioning_warnings

HOST_BCAST_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int)


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Rank's contiguous column block [c0, c1) (mirrors bse::shard_range)."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError("bad shard arguments")
    return n * rank // world, n * (rank + 1) // world


def make_host_bcast(group=None):
    """A host broadcast callback over a torch.distributed group: broadcasts
    ``nbytes`` at host address ``buf`` from ``root`` (returns 0 / 1)."""
    import torch
    import torch.distributed as dist

    def bcast(_ctx, buf, nbytes, root):
        try:
            if nbytes:
                arr = (C.c_uint8 * nbytes).from_address(buf)
                t = torch.frombuffer(arr, dtype=torch.uint8)
                dist.broadcast(t, src=dist.get_global_rank(group, root) if group is not None
                               else root, group=group)
            return 0
        except Exception:  # never raise through the C ABI
            return 1
    return bcast


def allgather_cols_host(a: np.ndarray, world: int, rank: int, bcast) -> np.ndarray:
    """Host mirror of bse::allgather_cols on a column-major numpy matrix
    (rows x n): every rank's column block is broadcast from its owner through
    the same callback the host transport uses.  Used by the CPU tests of the
    sharding logic."""
    n = a.shape[1]
    out = np.asfortranarray(a.copy())
    for r in range(world):
        c0, c1 = shard_range(n, world, r)
        if c1 > c0:
            blk = np.asfortranarray(out[:, c0:c1])
            if bcast(None, blk.ctypes.data, blk.nbytes, r) != 0:
                raise RuntimeError("host broadcast failed")
            out[:, c0:c1] = blk
    return out


# ---------------------------------------------------------------------------
# Block-cyclic column layout of the memory-distributed solve (csrc/dist.cuh,
# BcLayout): the 1 x Q grid of the 2-D block-cyclic family, tile nb.  Pure
# index arithmetic, mirrored here so callers (and the CPU tests) can scatter
# and gather matrices without the library.

def bc_owner(tile: int, world: int) -> int:
    """Rank owning global column tile ``tile``."""
    return tile % world


def bc_local_cols(n: int, nb: int, world: int, rank: int) -> np.ndarray:
    """Global column indices of ``rank``'s columns, in local order."""
    if n < 0 or nb < 1 or world < 1 or not 0 <= rank < world:
        raise ValueError("bad block-cyclic arguments")
    cols = [np.arange(t * nb, min((t + 1) * nb, n)) for t in range(rank, -(-n // nb), world)]
    return np.concatenate(cols) if cols else np.zeros(0, dtype=np.int64)


def bc_scatter(a: np.ndarray, nb: int, world: int, rank: int) -> np.ndarray:
    """This rank's columns of the global matrix ``a`` (rows x n)."""
    return a[:, bc_local_cols(a.shape[1], nb, world, rank)]


def bc_gather(blocks, n: int, nb: int) -> np.ndarray:
    """Global matrix from every rank's local columns (``blocks[r]``: rows x nloc_r)."""
    world = len(blocks)
    out = np.empty((blocks[0].shape[0], n), dtype=blocks[0].dtype)
    for r, blk in enumerate(blocks):
        out[:, bc_local_cols(n, nb, world, r)] = blk
    return out


class Communicator:
    """Owns a ``bse_comm`` handle of the C ABI (NCCL or host-staged)."""

    def __init__(self, handle, rank: int, world: int, keepalive=None):
        self._h = handle
        self.rank = rank
        self.world = world
        self._keep = keepalive

    @classmethod
    def nccl(cls, group=None):
        """NCCL communicator over the ranks of an initialised torch.distributed
        group (rank 0 creates the ncclUniqueId; the group carries it)."""
        import torch.distributed as dist
        lib = _lib.load()
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = C.create_string_buffer(128)
        if rank == 0 and lib.bse_comm_nccl_unique_id(uid) != _lib.BSE_OK:
            raise RuntimeError(f"ncclGetUniqueId failed: {_lib.last_error()}")
        box = [uid.raw if rank == 0 else None]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                   group=group)
        uid = C.create_string_buffer(box[0], 128)
        h = C.c_void_p()
        if lib.bse_comm_create_nccl(rank, world, uid, C.byref(h)) != _lib.BSE_OK:
            raise RuntimeError(f"NCCL communicator: {_lib.last_error()}")
        return cls(h, rank, world)

    @classmethod
    def host(cls, group=None):
        """Host-staged transport over a torch.distributed (gloo) group."""
        import torch.distributed as dist
        lib = _lib.load()
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        fn = HOST_BCAST_FN(make_host_bcast(group))
        h = C.c_void_p()
        if lib.bse_comm_create_host(rank, world, fn, None, C.byref(h)) != _lib.BSE_OK:
            raise RuntimeError(f"host communicator: {_lib.last_error()}")
        return cls(h, rank, world, keepalive=fn)

    @classmethod
    def solo(cls, rank: int, world: int):
        """Measurement-only transport: the kernels of rank ``rank`` of a
        ``world``-GPU solve on this GPU, with no exchange (not a solution)."""
        h = C.c_void_p()
        if _lib.load().bse_comm_create_solo(rank, world, C.byref(h)) != _lib.BSE_OK:
            raise RuntimeError(f"solo communicator: {_lib.last_error()}")
        return cls(h, rank, world)

    @property
    def handle(self):
        if self._h is None:
            raise RuntimeError("communicator is closed")
        return self._h

    def allgather_cols(self, t, ld: int, n: int):
        """Broadcast every rank's column block of a column-major device buffer."""
        st = _lib.load().bse_comm_allgather_cols_dev(self.handle, ptr(t), ld, n, stream_ptr(t.device))
        if st != _lib.BSE_OK:
            raise RuntimeError(f"allgather_cols failed: {_lib.last_error()}")

    def close(self):
        if self._h is not None:
            _lib.load().bse_comm_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve_pair_device_dist(comm: Communicator, Mt, ldm: int, Kt, ldk: int, n: int,
                           flags: int = 0, out=None):
    """Collective bse_solve_spd_pair_dist_dev: every rank passes the same
    (M, K); every rank returns (lam, X1, X2, ld) in full.  ``out`` may supply
    preallocated (lam, X1, X2, ld, work) buffers."""
    torch = require_cuda()
    lib = _lib.load()
    dev = Mt.device
    if out is None:
        X1, ld = colmajor_empty(n, n, dev)
        X2, _ = colmajor_empty(n, n, dev)
        lam = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
        wb = lib.bse_solve_workspace_bytes(n, flags)
        work = torch.empty(max(int(wb), 1), dtype=torch.uint8, device=dev)
    else:
        lam, X1, X2, ld, work = out
        wb = work.numel()
    info = _lib.BseInfo()
    st = lib.bse_solve_spd_pair_dist_dev(comm.handle, n, ptr(Mt), ldm, ptr(Kt), ldk, ptr(lam),
                                         ptr(X1), ld, ptr(X2), ld, ptr(work), wb, flags,
                                         stream_ptr(dev), C.byref(info))
    if st == _lib.BSE_NOT_POSITIVE_DEFINITE:
        err = NotPositiveDefinite(int(info.pivot_index), float(info.pivot_value),
                                  "A+B" if info.failed_factor == 1 else "A-B")
        err.failed_factor = int(info.failed_factor)
        raise err
    if st != _lib.BSE_OK:
        raise RuntimeError(f"bse_solve_spd_pair_dist_dev failed ({st}): {_lib.last_error()}")
    return lam[:n], X1, X2, ld


def bc_workspace_bytes(n: int, nb: int, world: int, rank: int, flags: int = 0):
    """(total, distributed, replicated) workspace bytes of one rank."""
    d, r = C.c_size_t(0), C.c_size_t(0)
    tot = _lib.load().bse_solve_bc_workspace_bytes(n, nb, world, rank, flags, C.byref(d), C.byref(r))
    return int(tot), int(d.value), int(r.value)


def solve_pair_device_bc(comm: Communicator, Mloc, ldm: int, Kloc, ldk: int, n: int, nb: int = 512,
                         flags: int = 0, out=None):
    """Collective bse_solve_spd_pair_bc_dev: every rank passes ITS columns of
    M and K (column-major device buffers, n rows) and gets lam (all n) and its
    columns of X1, X2 back: (lam, X1loc, X2loc, ld)."""
    torch = require_cuda()
    lib = _lib.load()
    dev = Mloc.device
    nloc = int(lib.bse_bc_local_cols(n, nb, comm.world, comm.rank))
    if nloc < 0:
        raise ValueError("bad block-cyclic arguments (nb must be a multiple of 64)")
    if out is None:
        X1, ld = colmajor_empty(n, nloc, dev)
        X2, _ = colmajor_empty(n, nloc, dev)
        lam = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
        wb = bc_workspace_bytes(n, nb, comm.world, comm.rank, flags)[0]
        work = torch.empty(max(wb, 1), dtype=torch.uint8, device=dev)
    else:
        lam, X1, X2, ld, work = out
        wb = work.numel()
    info = _lib.BseInfo()
    st = lib.bse_solve_spd_pair_bc_dev(comm.handle, n, nb, ptr(Mloc), ldm, ptr(Kloc), ldk, ptr(lam),
                                       ptr(X1), ld, ptr(X2), ld, ptr(work), wb, flags,
                                       stream_ptr(dev), C.byref(info))
    if st == _lib.BSE_NOT_POSITIVE_DEFINITE:
        err = NotPositiveDefinite(int(info.pivot_index), float(info.pivot_value),
                                  "A+B" if info.failed_factor == 1 else "A-B")
        err.failed_factor = int(info.failed_factor)
        raise err
    if st == _lib.BSE_NO_CONVERGENCE:
        from .types import ConvergenceError
        raise ConvergenceError(_lib.last_error())
    if st == _lib.BSE_SPECTRUM_NOT_POSITIVE:
        raise ValueError("all eigenvalues must be strictly positive")
    if st != _lib.BSE_OK:
        raise RuntimeError(f"bse_solve_spd_pair_bc_dev failed ({st}): {_lib.last_error()}")
    return lam[:n], X1, X2, ld


def solve_real_bc(op: BseOperator, comm: Communicator, nb: int = 512):
    """Memory-distributed ``solve_real`` (reference: solvers.py:80-109): every
    rank uploads only its block-cyclic columns of A+B and A-B and returns
    (lambda_plus, x1_local, x2_local, global_columns): all n eigenvalues and
    this rank's columns of X1, X2 (float64, n x nloc)."""
    if op.kind != "real":
        raise ValueError("solve_real requires an operator of kind 'real'")
    n = op.n
    torch = require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    cols = bc_local_cols(n, nb, comm.world, comm.rank)
    a, b = op.a.real, op.b.real
    Mloc, ldm = to_device_colmajor((a + b)[:, cols], dev)
    Kloc, ldk = to_device_colmajor((a - b)[:, cols], dev)
    lam, X1, X2, _ = solve_pair_device_bc(comm, Mloc, ldm, Kloc, ldk, n, nb)
    return (lam.cpu().numpy(), from_device_colmajor(X1, n, len(cols)),
            from_device_colmajor(X2, n, len(cols)), cols)


def solve_real(op: BseOperator, comm: Communicator) -> PositiveEigensystem:
    """Sharded ``solve_real`` (reference: solvers.py:80-109): called by every
    rank of ``comm`` with the same operator; every rank returns the full
    PositiveEigensystem."""
    if op.kind != "real":
        raise ValueError("solve_real requires an operator of kind 'real'")
    n = op.n
    if n == 0:
        return PositiveEigensystem(lambda_plus=np.zeros(0), x1=np.zeros((0, 0)), x2=np.zeros((0, 0)))
    torch = require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    a, b = op.a.real, op.b.real
    Mt, ldm = to_device_colmajor(a + b, dev)
    Kt, ldk = to_device_colmajor(a - b, dev)
    lam, X1, X2, _ = solve_pair_device_dist(comm, Mt, ldm, Kt, ldk, n)
    lam_h = lam.cpu().numpy()
    x1 = from_device_colmajor(X1, n, n)
    x2 = from_device_colmajor(X2, n, n)
    return PositiveEigensystem(lambda_plus=lam_h, x1=x1.astype(np.complex128),
                               x2=x2.astype(np.complex128), warnings=conditioning_warnings(lam_h))
