"""Block-cyclic multi-GPU pivoted LTL^T (config 5).

The reference has no distributed path; this is ``ltlt_blk_piv``
(``blocked.py:303-363``) over G ranks with a 1-D block-cyclic column
distribution: column block j = [j*nbd, (j+1)*nbd) lives in the HBM of rank
j % G.  One process per GPU (``torch.distributed`` for the plumbing).

B200 design: every rank maps ALL column blocks -- its own and its peers' --
into ONE virtual address range with CUDA VMM (physical allocations exported
as POSIX fds and imported by the peers), so the work matrix is a single
column-major array on every GPU and the kernels reach remote columns with
plain NVLink loads and stores.  The per-panel exchange of §8e (pivot-column
fetches, the panel broadcast, the cross-owner interchanges) is therefore not
a sequence of messages: the panel runner gathers each pivot column straight
from its owner's HBM, and every rank reads the finished panel block to pack
its trailing-update operands.  The only collective is a stream-ordered
barrier twice per panel (NCCL one-word all-reduce, native, or a host barrier
for several ranks sharing one device).

Two ways to run it:

* ``group`` = an initialised process group, one rank per GPU (``torchrun``);
* ``virtual_ranks=G`` in one process on one device: G physical allocations on
  the same GPU, the same block-cyclic mapping, the same kernels with every
  rank's column filter -- the single-device emulation used by the tests.

Nothing here runs on the CPU; the compute is ``skl_ltlt_blk_piv_dist``.
"""

from __future__ import annotations

import ctypes as C
import os
import secrets
import socket
import threading
import time

import numpy as np

from . import _capi
from . import device as dv
from .core import InvalidVariant

DEFAULT_NBD = 512


# ---------------------------------------------------------------------------
# block-cyclic bookkeeping (pure host logic)
# ---------------------------------------------------------------------------
class BlockCyclic:
    """Column block j = [j*nbd, min(n, (j+1)*nbd)) is owned by rank j % G (one
    physical allocation per block on that rank)."""

    def __init__(self, n, nbd, nranks):
        if n < 1 or nbd < 1 or nranks < 1:
            raise ValueError("n, nbd, nranks must be >= 1")
        self.n, self.nbd, self.G = int(n), int(nbd), int(nranks)
        self.nblocks = (self.n + self.nbd - 1) // self.nbd

    def owner(self, col):
        return (int(col) // self.nbd) % self.G

    def blocks_of(self, rank):
        return list(range(rank, self.nblocks, self.G))

    def nblocks_of(self, rank):
        return len(self.blocks_of(rank))

    def columns_of(self, rank):
        cols = [np.arange(j * self.nbd, min(self.n, (j + 1) * self.nbd)) for j in self.blocks_of(rank)]
        return np.concatenate(cols) if cols else np.zeros(0, dtype=np.int64)

    def block_range(self, j):
        return j * self.nbd, min(self.n, (j + 1) * self.nbd)


def padded_ld(n, nbd, gran):
    """Smallest ld >= n with nbd*ld*8 a multiple of the VMM granularity, so
    every column block is an exact number of mapping granules."""
    unit = gran // np.gcd(gran, nbd * 8)
    return int(-(-n // unit) * unit)


def owner_table(n, cbase, nbd, nranks, rank):
    """The column-filtered GEMM's owned-tile table (skl_dist_owner_table)."""
    lib = _capi.load()
    nt = (n + 127) // 128
    tab = (C.c_int * (2 + 4 * nt))()
    _capi.check(lib.skl_dist_owner_table(n, cbase, nbd, nranks, rank, tab, len(tab)), "dist_owner_table")
    m = tab[0]
    rows = [(tab[2 + 4 * c], tab[3 + 4 * c], tab[4 + 4 * c]) for c in range(m)]
    assert all(tab[5 + 4 * c] == tab[2 + 4 * c] for c in range(m))  # lower tiles: rows start at the diagonal
    return tab[1], rows


# ---------------------------------------------------------------------------
# device plumbing
# ---------------------------------------------------------------------------
class _DevPtr:
    """__cuda_array_interface__ over a raw device address (torch.as_tensor view)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def colmajor_view(ptr, rows, cols, ld, typestr="<f8"):
    t = dv.require_cuda()
    return t.as_tensor(_DevPtr(ptr, (cols, ld), typestr), device="cuda").t()[:rows, :cols]


def vector_view(ptr, length, typestr):
    t = dv.require_cuda()
    return t.as_tensor(_DevPtr(ptr, (length,), typestr), device="cuda")


def _vmm_check(rc, what):
    if rc != _capi.SKL_OK:
        raise _capi.NativeError(f"{what} failed (status {rc}, CUresult {_capi.load().skl_vmm_last_result()})")


class _Phys:
    """One VMM physical allocation (owned here or imported from a peer)."""

    def __init__(self, handle, nbytes, fd=-1):
        self.handle, self.nbytes, self.fd = handle, nbytes, fd


def _create_phys(nbytes, device, exportable):
    lib = _capi.load()
    h = C.c_ulonglong(0)
    _vmm_check(lib.skl_vmm_create(nbytes, device, 1 if exportable else 0, C.byref(h)), "cuMemCreate")
    fd = -1
    if exportable:
        f = C.c_int(-1)
        _vmm_check(lib.skl_vmm_export_fd(h.value, C.byref(f)), "cuMemExportToShareableHandle")
        fd = f.value
    return _Phys(h.value, nbytes, fd)


def _import_phys(fd, nbytes):
    lib = _capi.load()
    h = C.c_ulonglong(0)
    _vmm_check(lib.skl_vmm_import_fd(fd, C.byref(h)), "cuMemImportFromShareableHandle")
    os.close(fd)
    return _Phys(h.value, nbytes)


class _Mapping:
    """A reserved VA range with (offset, bytes, phys, phys_offset) pieces mapped."""

    def __init__(self, nbytes, gran, device):
        lib = _capi.load()
        va = C.c_ulonglong(0)
        _vmm_check(lib.skl_vmm_reserve(nbytes, gran, C.byref(va)), "cuMemAddressReserve")
        self.va, self.nbytes, self.device, self.pieces = va.value, nbytes, device, []

    def map(self, off, nbytes, phys, phys_off):
        _vmm_check(_capi.load().skl_vmm_map(self.va + off, nbytes, phys.handle, phys_off, self.device), "cuMemMap")
        self.pieces.append((off, nbytes))

    def close(self):
        lib = _capi.load()
        for off, nb in self.pieces:
            lib.skl_vmm_unmap(self.va + off, nb)
        self.pieces = []
        if self.va:
            lib.skl_vmm_free_va(self.va, self.nbytes)
            self.va = 0


def _recv_exact(sock, nbytes):
    buf = b""
    while len(buf) < nbytes:
        part = sock.recv(nbytes - len(buf))
        if not part:
            raise ConnectionError("peer closed the fd exchange")
        buf += part
    return buf


def exchange_fds(my_fds, rank, world, group=None, token=None):
    """All-to-all exchange of file descriptors between the ranks of a process
    group over abstract Unix sockets (SCM_RIGHTS).  Returns {peer: [fds]}."""
    import torch.distributed as tdist
    if token is None:
        obj = [secrets.token_hex(8) if rank == 0 else None]
        tdist.broadcast_object_list(obj, src=0, group=group)
        token = obj[0]
    name = f"\0skl-b200-{token}-{{}}"
    srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    srv.bind(name.format(rank))
    srv.listen(max(world - 1, 1))
    tdist.barrier(group=group)  # every rank listens before anyone connects

    def serve():
        for _ in range(world - 1):
            conn, _addr = srv.accept()
            with conn:
                conn.recv(1)
                conn.sendall(np.int32(len(my_fds)).tobytes())
                for k in range(0, len(my_fds), 200):   # SCM_RIGHTS carries <= 253 fds per message
                    socket.send_fds(conn, [b"f"], list(my_fds[k:k + 200]))
                    conn.recv(1)

    th = threading.Thread(target=serve, daemon=True)
    th.start()
    got = {}
    for q in range(world):
        if q == rank:
            continue
        with socket.socket(socket.AF_UNIX, socket.SOCK_STREAM) as c:
            for _attempt in range(200):
                try:
                    c.connect(name.format(q))
                    break
                except (ConnectionRefusedError, FileNotFoundError):
                    time.sleep(0.01)
            c.sendall(b"x")
            count = int(np.frombuffer(_recv_exact(c, 4), dtype=np.int32)[0])
            fds = []
            while len(fds) < count:
                _msg, part, _flags, _addr = socket.recv_fds(c, 1, 200)
                fds.extend(part)
                c.sendall(b"k")
            got[q] = fds
    th.join()
    srv.close()
    tdist.barrier(group=group)
    return got


# ---------------------------------------------------------------------------
# the distributed factorization
# ---------------------------------------------------------------------------
class DistLTLT:
    """Distributed work matrix + factorization state for one (n, nb, variant).

    ``group``: process group of G ranks (one per GPU); or ``virtual_ranks=G``
    (single process, one device).  ``barrier``: "nccl" (native one-word
    all-reduce on the stream) or "host" (stream sync + process-group barrier;
    needed when several ranks share one device, where NCCL refuses).
    """

    def __init__(self, n, b=DEFAULT_NBD, fused="var1", nbd=None, group=None, virtual_ranks=None, barrier="nccl"):
        if fused not in _capi.VARIANT_CODES:
            raise InvalidVariant(f"fused must be one of {tuple(_capi.VARIANT_CODES)}, got {fused!r}")
        if b < 1:
            raise ValueError("b >= 1 required")
        t = dv.require_cuda()
        lib = _capi.load()
        if not lib.skl_vmm_available():
            raise _capi.NativeUnavailable("CUDA VMM entry points unavailable")
        self.n, self.b, self.fused = int(n), int(b), fused
        self.variant = _capi.VARIANT_CODES[fused]
        if self.n < 2:
            raise ValueError("the distributed driver needs n >= 2")
        self.device = t.cuda.current_device()
        if group is not None or virtual_ranks is None:
            import torch.distributed as tdist
            self.group = group
            self.G = tdist.get_world_size(group)
            self.rank = tdist.get_rank(group)
            self.rank_lo, self.rank_hi = self.rank, self.rank + 1
            self.multi = self.G > 1
        else:
            self.group = None
            self.G = int(virtual_ranks)
            self.rank, self.rank_lo, self.rank_hi = 0, 0, self.G
            self.multi = False
        self.nbd = int(nbd) if nbd else DEFAULT_NBD
        self.bc = BlockCyclic(self.n, self.nbd, self.G)
        gran = C.c_size_t(0)
        _vmm_check(lib.skl_vmm_granularity(self.device, C.byref(gran)), "granularity")
        self.gran = gran.value
        self.ld = padded_ld(self.n, self.nbd, self.gran)
        self.block_bytes = self.nbd * self.ld * 8
        self.shared_bytes = lib.skl_ltlt_dist_shared_size(self.n, self.b, self.variant)
        if self.shared_bytes == 0:
            raise InvalidVariant("configuration not supported by the GPU panel kernels")
        self.shared_bytes = -(-self.shared_bytes // self.gran) * self.gran
        nloc = self.rank_hi - self.rank_lo
        self.ws_bytes = lib.skl_ltlt_dist_workspace_size(self.n, self.b, self.variant, nloc)
        off_tau, off_piv = C.c_size_t(0), C.c_size_t(0)
        _capi.check(lib.skl_ltlt_dist_offsets(self.n, self.b, self.variant, C.byref(off_tau), C.byref(off_piv),
                                              None, None), "dist_offsets")
        self.off_tau, self.off_piv = off_tau.value, off_piv.value
        self._build_mappings()
        self.workspace = t.empty(self.ws_bytes, dtype=t.uint8, device="cuda")
        self._barrier_kind = barrier
        self._barrier_ctx = None
        self._cb = None
        if self.multi:
            self._setup_barrier(barrier)

    # -- memory ----------------------------------------------------------------
    def _build_mappings(self):
        # cuMemMap maps a physical allocation from offset 0 only, so every column
        # block of W and L is its own allocation (exported as its own fd)
        G, nb = self.G, self.bc.nblocks
        span = nb * self.block_bytes
        phys = {}  # block -> (W phys, L phys)
        for r in range(self.rank_lo, self.rank_hi):
            for j in self.bc.blocks_of(r):
                phys[j] = (_create_phys(self.block_bytes, self.device, self.multi),
                           _create_phys(self.block_bytes, self.device, self.multi))
        shared = _create_phys(self.shared_bytes, self.device, self.multi) if self.rank_lo == 0 else None
        if self.multi:
            mine = self.bc.blocks_of(self.rank)
            my = [f for j in mine for f in (phys[j][0].fd, phys[j][1].fd)]
            my += [shared.fd] if shared is not None else []
            got = exchange_fds(my, self.rank, G, self.group)
            for q, fds in got.items():
                blocks = self.bc.blocks_of(q)
                for i, j in enumerate(blocks):
                    phys[j] = (_import_phys(fds[2 * i], self.block_bytes), _import_phys(fds[2 * i + 1], self.block_bytes))
                if q == 0:
                    shared = _import_phys(fds[2 * len(blocks)], self.shared_bytes)
            for f in my:
                os.close(f)
        self._phys = [p for pair in phys.values() for p in pair] + [shared]
        self.W = _Mapping(span, self.gran, self.device)
        self.L = _Mapping(span, self.gran, self.device)
        for j in range(nb):
            self.W.map(j * self.block_bytes, self.block_bytes, phys[j][0], 0)
            self.L.map(j * self.block_bytes, self.block_bytes, phys[j][1], 0)
        self.S = _Mapping(self.shared_bytes, self.gran, self.device)
        self.S.map(0, self.shared_bytes, shared, 0)

    def w_view(self):
        return colmajor_view(self.W.va, self.n, self.n, self.ld)

    def l_view(self):
        return colmajor_view(self.L.va, self.n, self.n, self.ld)

    def tau_view(self):
        return vector_view(self.S.va + self.off_tau, self.n - 1, "<f8")

    def piv_view(self):
        return vector_view(self.S.va + self.off_piv, self.n, "<i8")

    # -- barrier -----------------------------------------------------------------
    def _setup_barrier(self, kind):
        import torch.distributed as tdist
        lib = _capi.load()
        if kind == "nccl":
            if not lib.skl_nccl_available():
                raise _capi.NativeUnavailable("libnccl.so.2 not loadable")
            uid = (C.c_ubyte * 128)()
            if self.rank == 0:
                _capi.check(lib.skl_nccl_unique_id(uid, 128), "ncclGetUniqueId")
            obj = [bytes(uid)]
            tdist.broadcast_object_list(obj, src=0, group=self.group)
            uid = (C.c_ubyte * 128).from_buffer_copy(obj[0])
            ctx = C.c_void_p(0)
            _capi.check(lib.skl_nccl_barrier_create(self.G, self.rank, uid, C.byref(ctx)), "ncclCommInitRank")
            self._barrier_ctx = ctx.value
            self._barrier_fn = C.cast(lib.skl_nccl_barrier, C.c_void_p).value
        elif kind == "host":
            import torch
            group = self.group

            def host_barrier(_ctx, stream):
                try:
                    torch.cuda.ExternalStream(stream).synchronize() if stream else torch.cuda.synchronize()
                    tdist.barrier(group=group)
                    return 0
                except Exception:  # noqa: BLE001 -- reported as a C status
                    return 1

            self._cb = _capi.BARRIER_FN(host_barrier)
            self._barrier_fn = C.cast(self._cb, C.c_void_p).value
        else:
            raise ValueError(f"barrier must be 'nccl' or 'host', got {kind!r}")

    # -- compute -----------------------------------------------------------------
    def load_input(self, x):
        """Copy this process's column blocks of X (full n x n: numpy F-order or a
        column-major CUDA tensor; only the strict lower triangle is used) into W."""
        t = dv.require_cuda()
        W = self.w_view()
        for r in range(self.rank_lo, self.rank_hi):
            for j in self.bc.blocks_of(r):
                c0, c1 = self.bc.block_range(j)
                src = x[:, c0:c1]
                if isinstance(src, np.ndarray):
                    src = t.from_numpy(np.ascontiguousarray(src.T)).to("cuda").t()
                W[:, c0:c1].copy_(src)

    def factorize(self, stream=None):
        """Run skl_ltlt_blk_piv_dist on the current W (stream-ordered, no host sync
        except the host-barrier mode).  Returns (L view, tau view, piv view)."""
        lib = _capi.load()
        fn = C.cast(C.c_void_p(self._barrier_fn), _capi.BARRIER_FN) if self.multi else None
        st = lib.skl_ltlt_blk_piv_dist(self.n, self.b, self.variant, self.nbd, self.G, self.rank_lo, self.rank_hi,
                                       self.W.va, self.ld, self.L.va, self.ld, self.S.va,
                                       self.workspace.data_ptr(), self.ws_bytes, fn,
                                       self._barrier_ctx, dv.stream_ptr(stream))
        _capi.check(st, "ltlt_blk_piv_dist")
        return self.l_view(), self.tau_view(), self.piv_view()

    def close(self):
        lib = _capi.load()
        for m in ("W", "L", "S"):
            mp = getattr(self, m, None)
            if mp is not None:
                mp.close()
        for p in getattr(self, "_phys", []):
            if p is not None:
                lib.skl_vmm_release(p.handle)
        self._phys = []
        if self._barrier_ctx and self._barrier_kind == "nccl":
            lib.skl_nccl_barrier_destroy(self._barrier_ctx)
            self._barrier_ctx = None


def ltlt_blk_piv_dist(x, b=DEFAULT_NBD, fused="var1", nbd=None, group=None, virtual_ranks=None, barrier="nccl"):
    """Distributed pivoted LTL^T of the full X (numpy or column-major CUDA tensor,
    identical on every rank).  Returns (ctx, L view, tau, piv): L is the global
    block-cyclic "ones" buffer (only this process's columns are written; other
    columns are readable over NVLink), tau/piv are the shared vectors.  Call
    ``ctx.close()`` when the views are no longer needed."""
    n = int(x.shape[0])
    ctx = DistLTLT(n, b, fused, nbd, group=group, virtual_ranks=virtual_ranks, barrier=barrier)
    ctx.load_input(x)      # same stream: the driver's first barrier orders every rank's copies
    L, tau, piv = ctx.factorize()
    return ctx, L, tau, piv
