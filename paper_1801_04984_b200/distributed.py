"""Multi-GPU slab block solve through the library (DESIGN.md section 6,
SURVEY.md 8(e)): one process per GPU, strips of cell rows per rank. The
operator halo exchange, the rank-ordered Krylov reductions, the substructured
exact inner solves and the GMRES loop all run inside libporodg_b200
(csrc/dist.cu, pdg_dblock_*); this module only creates the communicator:

- `nccl_comm`: NCCL, the unique id distributed over torch.distributed;
- `host_comm`: host-staged collectives through torch.distributed callbacks
  (gloo), so several ranks can share one GPU in the tests without any kernel
  waiting on another rank's kernel.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check, lib
from .solver import context


class TriSolver:
    """pdg_tri_*: exact block-tridiagonal solve of a host CSR on the device (SPD:
    twisted Cholesky; symmetric=False: twisted block LU)."""

    def __init__(self, A, block_sizes, perm=None, allow_local=True, device: int = 0, symmetric=True):
        import scipy.sparse as sp

        A = sp.csr_matrix(A)
        A.sort_indices()
        self.n = A.shape[0]
        off = np.ascontiguousarray(A.indptr, np.int32)
        idx = np.ascontiguousarray(A.indices, np.int32)
        val = np.ascontiguousarray(A.data, np.float64)
        csr = _lib.CSR(self.n, self.n, len(val), off.ctypes.data_as(C.POINTER(C.c_int)),
                       idx.ctypes.data_as(C.POINTER(C.c_int)), val.ctypes.data_as(_lib.DP))
        bs = np.ascontiguousarray(block_sizes, np.int32)
        pm = None if perm is None else np.ascontiguousarray(perm, np.int32)
        h = C.c_void_p()
        check(lib().pdg_tri_create(context(device), C.byref(csr), None if pm is None else pm.ctypes.data_as(_lib.IP),
                                   bs.ctypes.data_as(_lib.IP), len(bs),
                                   (1 if allow_local else 0) | (0 if symmetric else 2), C.byref(h)))
        self._h = h

    def solve(self, b):
        """b: (n,) or (n, k) device tensor (k <= 2 per library call)."""
        import torch

        b2 = b.reshape(self.n, -1)
        out = torch.empty_like(b2)
        for c0 in range(0, b2.shape[1], 2):
            cols = b2[:, c0:c0 + 2].t().contiguous()  # column-major: rhs after rhs
            x = torch.empty_like(cols)
            torch.cuda.synchronize()
            check(lib().pdg_tri_solve_device(self._h, cols.data_ptr(), x.data_ptr(), cols.shape[0]))
            out[:, c0:c0 + 2] = x.t()
        return out.reshape(b.shape)

    def __del__(self):
        if getattr(self, "_h", None) and _lib._lib is not None:
            _lib._lib.pdg_tri_destroy(self._h)
            self._h = None



_HOST_AG = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_longlong)
_HOST_EX = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.POINTER(C.c_double)),
                       C.POINTER(C.c_longlong), C.POINTER(C.POINTER(C.c_double)), C.POINTER(C.c_longlong))


class LibComm:
    """A library communicator (pdg_comm) of this rank."""

    def __init__(self, handle, rank, nranks, keep=()):
        self._h, self.rank, self.nranks, self._keep = handle, rank, nranks, keep

    def __del__(self):
        if getattr(self, "_h", None) and _lib._lib is not None:
            _lib._lib.pdg_comm_destroy(self._h)
            self._h = None


def nccl_comm(dist, rank: int, nranks: int, device: int = 0) -> LibComm:
    """NCCL communicator: rank 0 makes the unique id, torch.distributed broadcasts it.
    torch is imported first so that the library uses torch's NCCL (csrc/dist.cu)."""
    import torch

    idb = (C.c_ubyte * 128)()
    if rank == 0:
        check(lib().pdg_nccl_unique_id(idb))
    if nranks > 1:
        t = torch.tensor(list(bytes(idb)), dtype=torch.uint8)
        if dist.get_backend() == "nccl":
            t = t.cuda(device)
        dist.broadcast(t, 0)
        idb = (C.c_ubyte * 128)(*t.cpu().tolist())
    h = C.c_void_p()
    check(lib().pdg_comm_create_nccl(context(device), nranks, rank, idb, C.byref(h)))
    return LibComm(h, rank, nranks)


def host_comm(dist, rank: int, nranks: int, device: int = 0) -> LibComm:
    """Host-staged communicator: the library calls back into torch.distributed (gloo,
    CPU tensors) for the all-gathers and the neighbour exchanges (batched p2p)."""
    import torch

    def allgather(_u, send, recv, count):
        try:
            src = torch.from_numpy(np.ctypeslib.as_array(send, shape=(max(count, 1),))[:count].copy())
            bufs = [torch.empty(count, dtype=torch.float64) for _ in range(nranks)]
            dist.all_gather(bufs, src)
            out = np.ctypeslib.as_array(recv, shape=(max(count * nranks, 1),))
            for r, b in enumerate(bufs):
                out[r * count:(r + 1) * count] = b.numpy()
            return 0
        except Exception:  # pragma: no cover - reported as a library error
            return 1

    def exchange(_u, npeers, peers, send, scount, recv, rcount):
        try:
            ops, rbufs = [], []
            for i in range(npeers):
                if scount[i]:
                    s_ = torch.from_numpy(np.ctypeslib.as_array(send[i], shape=(scount[i],)).copy())
                    ops.append(dist.P2POp(dist.isend, s_, peers[i]))
                rb = torch.empty(rcount[i], dtype=torch.float64)
                rbufs.append(rb)
                if rcount[i]:
                    ops.append(dist.P2POp(dist.irecv, rb, peers[i]))
            if ops:
                for req in dist.batch_isend_irecv(ops):
                    req.wait()
            for i in range(npeers):
                if rcount[i]:
                    np.ctypeslib.as_array(recv[i], shape=(rcount[i],))[:] = rbufs[i].numpy()
            return 0
        except Exception:  # pragma: no cover
            return 1

    ag, ex = _HOST_AG(allgather), _HOST_EX(exchange)
    h = C.c_void_p()
    check(lib().pdg_comm_create_host(context(device), nranks, rank, C.cast(ag, C.c_void_p), C.cast(ex, C.c_void_p),
                                     None, C.byref(h)))
    return LibComm(h, rank, nranks, keep=(ag, ex))


class DistributedBlock:
    """pdg_dblock: the transformed slab block (m components, Theta, tau; the
    preconditioner's lambda = Theta[0, 0], slab.hpp:220-227) solved by GMRES
    across the ranks of `comm`; vectors are this rank's owned rows (global
    indices in `owned`)."""

    def __init__(self, ops, comm: LibComm, theta, tau, opt=None):
        from . import solver as S

        opt = opt or S.SolveOptions()
        self.theta = np.ascontiguousarray(np.atleast_2d(theta), np.float64)
        self.m = self.theta.shape[0]
        self.comm = comm
        o = opt.to_struct()
        h = C.c_void_p()
        check(lib().pdg_dblock_create(ops._h, comm._h, self.m, self.theta.ctypes.data_as(_lib.DP), tau,
                                      float(self.theta[0, 0]), C.byref(o), C.byref(h)))
        self._h, self._ops, self.max_iter = h, ops, opt.gmres.max_iter
        no, ng = C.c_longlong(), C.c_longlong()
        check(lib().pdg_dblock_rows(self._h, C.byref(no), C.byref(ng)))
        self.n_owned, self.n_global = no.value, ng.value
        rows = np.empty(self.n_owned, np.int64)
        check(lib().pdg_dblock_owned_rows(self._h, rows.ctypes.data_as(_lib.LLP)))
        self.owned = rows

    def solve_device(self, rhs_ptr: int, x_ptr: int):
        from .solver import _report, _to_report

        rep, hist = _report(self.max_iter + 2)
        check(lib().pdg_dblock_solve_device(self._h, rhs_ptr, x_ptr, C.byref(rep)))
        return _to_report(rep, hist)

    def solve(self, rhs_owned):
        """rhs_owned: this rank's rows (host array). Returns (x_owned, report)."""
        import torch

        b = torch.as_tensor(np.ascontiguousarray(rhs_owned, np.float64), device="cuda")
        x = torch.empty_like(b)
        torch.cuda.synchronize()
        rep = self.solve_device(b.data_ptr(), x.data_ptr())
        return x.cpu().numpy(), rep

    def apply(self, x_owned):
        import torch

        b = torch.as_tensor(np.ascontiguousarray(x_owned, np.float64), device="cuda")
        y = torch.empty_like(b)
        torch.cuda.synchronize()
        check(lib().pdg_dblock_apply_device(self._h, b.data_ptr(), y.data_ptr()))
        return y.cpu().numpy()

    def precondition(self, r_owned):
        import torch

        b = torch.as_tensor(np.ascontiguousarray(r_owned, np.float64), device="cuda")
        z = torch.empty_like(b)
        torch.cuda.synchronize()
        check(lib().pdg_dblock_precondition_device(self._h, b.data_ptr(), z.data_ptr()))
        return z.cpu().numpy()

    def __del__(self):
        if getattr(self, "_h", None) and _lib._lib is not None:
            _lib._lib.pdg_dblock_destroy(self._h)
            self._h = None
