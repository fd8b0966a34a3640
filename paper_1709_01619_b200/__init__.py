"""paper_1709_01619_b200 -- B200 (sm_100a) hot path of arXiv 1709.01619.

Thin ctypes binding of libhom2d.so (include/hom2d.h).  Argument marshalling
only: every step of the residual / RK / dt / error path runs in the library's
CUDA kernels.  PyTorch provides device memory (the workspace), streams and the
process group used to broadcast the NCCL id.  There is no CPU fallback: if the
extension is missing, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# HOM2D_LIB selects an alternative in-tree build (A/B timing of kernel variants)
LIB_PATH = os.environ.get("HOM2D_LIB") or os.path.join(HERE, "libhom2d.so")

FV, CPR, DG, NDG, SD = 0, 1, 2, 3, 4
PERIODIC, TRANSMISSIVE = 0, 1
VORTEX, SHOCK = 0, 1
METHODS = {"fv": FV, "cpr": CPR, "dg": DG, "ndg": NDG, "sd": SD}
STATUS = {0: "OK", 1: "ERR_ARG", 2: "ERR_MESH", 3: "ERR_ORDER", 4: "ERR_NONPHYSICAL", 5: "ERR_CUDA",
          6: "ERR_NCCL", 7: "ERR_NOMEM", 8: "ERR_STATE"}

# every symbol include/hom2d.h declares
EXPORTS = ["hom2d_strip_plan", "hom2d_workspace_bytes", "hom2d_nccl_unique_id", "hom2d_create", "hom2d_local_extent",
           "hom2d_set_state", "hom2d_get_state", "hom2d_init_case", "hom2d_residual", "hom2d_residual_strip", "hom2d_limit",
           "hom2d_compute_dt", "hom2d_step", "hom2d_error", "hom2d_time", "hom2d_decisions", "hom2d_decision_map",
           "hom2d_launch_count", "hom2d_stage_timing", "hom2d_stage_time", "hom2d_last_error", "hom2d_destroy",
           "hom2d_peer_id", "hom2d_peer_connect"]


class Hom2dError(RuntimeError):
    def __init__(self, status, msg=""):
        self.status = status
        super().__init__(f"hom2d {STATUS.get(status, status)}: {msg}")


class NonPhysicalState(Hom2dError):
    pass


class Config(C.Structure):
    _fields_ = [
        ("nx", C.c_int32), ("ny", C.c_int32),
        ("xmin", C.c_double), ("xmax", C.c_double), ("ymin", C.c_double), ("ymax", C.c_double),
        ("bc", C.c_int32), ("method", C.c_int32), ("k", C.c_int32),
        ("gamma", C.c_double), ("cfl", C.c_double),
        ("limiter", C.c_int32), ("limiter_eps", C.c_double),
        ("cpr_chain_rule", C.c_int32), ("record_decisions", C.c_int32),
        ("limiter_per_step", C.c_int32), ("limiter_all_vars", C.c_int32), ("fv_unlimited", C.c_int32),
        ("limiter_characteristic", C.c_int32), ("fv_error_recon", C.c_int32), ("dg_overintegrate", C.c_int32),
    ]


class StripPlan(C.Structure):
    _fields_ = [("row0", C.c_int32), ("nrows", C.c_int32), ("ghost_rows", C.c_int32),
                ("peer_lo", C.c_int32), ("peer_hi", C.c_int32), ("has_lo", C.c_int32), ("has_hi", C.c_int32),
                ("row_values", C.c_int64)]


class PeerId(C.Structure):
    _fields_ = [("ipc", C.c_uint8 * 64), ("offset", C.c_uint64), ("rank", C.c_int32), ("device", C.c_int32)]


class Dist(C.Structure):
    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32), ("device", C.c_int32),
                ("nccl_id", C.c_void_p), ("cuda_stream", C.c_void_p)]


_lib = None


def load(path: str = LIB_PATH):
    """Load libhom2d.so (torch is imported first so that its NCCL is the one in use)."""
    global _lib
    if _lib is not None:
        return _lib
    import torch  # noqa: F401  (device memory, streams; loads the NCCL the library links)
    if not os.path.exists(path):
        raise RuntimeError(f"libhom2d.so not built ({path}); run `python -m paper_1709_01619_b200.build`")
    L = C.CDLL(path)
    i32, i64, d, vp, P = C.c_int32, C.c_int64, C.c_double, C.c_void_p, C.POINTER
    L.hom2d_strip_plan.argtypes = [P(Config), i32, i32, P(StripPlan)]
    L.hom2d_workspace_bytes.argtypes = [P(Config), P(Dist), P(C.c_size_t)]
    L.hom2d_nccl_unique_id.argtypes = [vp]
    L.hom2d_create.argtypes = [P(Config), P(Dist), vp, C.c_size_t, P(vp)]
    L.hom2d_local_extent.argtypes = [vp, P(i32), P(i32), P(i64)]
    L.hom2d_set_state.argtypes = [vp, vp, i64, i32, d]
    L.hom2d_get_state.argtypes = [vp, vp, i64, i32]
    L.hom2d_init_case.argtypes = [vp, i32]
    L.hom2d_residual.argtypes = [vp, vp, vp]
    L.hom2d_residual_strip.argtypes = [vp, vp, vp, vp, vp]
    L.hom2d_limit.argtypes = [vp]
    L.hom2d_compute_dt.argtypes = [vp, P(d)]
    L.hom2d_step.argtypes = [vp, i32, d, P(d), P(i64)]
    L.hom2d_error.argtypes = [vp, i32, i32, P(d), P(d), P(d)]
    L.hom2d_time.argtypes = [vp, P(d)]
    L.hom2d_decisions.argtypes = [vp, vp]
    L.hom2d_decision_map.argtypes = [vp, vp, i64]
    L.hom2d_launch_count.argtypes = [vp]
    L.hom2d_launch_count.restype = i64
    L.hom2d_stage_timing.argtypes = [vp, i32]
    L.hom2d_stage_time.argtypes = [vp, P(d), P(i64)]
    L.hom2d_last_error.argtypes = [vp]
    L.hom2d_last_error.restype = C.c_char_p
    L.hom2d_peer_id.argtypes = [vp, P(PeerId)]
    L.hom2d_peer_connect.argtypes = [vp, P(PeerId), P(PeerId)]
    L.hom2d_destroy.argtypes = [vp]
    L.hom2d_destroy.restype = None
    for name in EXPORTS:
        if name not in ("hom2d_launch_count", "hom2d_last_error", "hom2d_destroy"):
            getattr(L, name).restype = C.c_int
    _lib = L
    return L


def make_config(nx, ny, method="cpr", k=1, bc=PERIODIC, box=(-5.0, 5.0, -5.0, 5.0), gamma=1.4, cfl=0.24,
                limiter=0, limiter_eps=1e-3, cpr_chain_rule=1, record_decisions=0, limiter_per_step=0,
                limiter_all_vars=0, fv_unlimited=0, limiter_characteristic=0, fv_error_recon=0,
                dg_overintegrate=0) -> Config:
    m = METHODS[method] if isinstance(method, str) else int(method)
    return Config(nx, ny, box[0], box[1], box[2], box[3], bc, m, k, gamma, cfl, limiter, limiter_eps,
                  cpr_chain_rule, record_decisions, limiter_per_step, limiter_all_vars, fv_unlimited,
                  limiter_characteristic, fv_error_recon, dg_overintegrate)


def strip_plan(cfg: Config, rank: int, nranks: int) -> StripPlan:
    """Host-only y-strip partition and halo plan of one rank (no CUDA)."""
    out = StripPlan()
    st = load().hom2d_strip_plan(C.byref(cfg), int(rank), int(nranks), C.byref(out))
    if st:
        raise Hom2dError(st, "strip_plan")
    return out


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = load().hom2d_nccl_unique_id(buf)
    if st:
        raise Hom2dError(st, "ncclGetUniqueId")
    return buf.raw


class Solver:
    """One hom2d handle: a strip of the grid on one GPU (all of it when nranks == 1)."""

    def __init__(self, cfg: Config, rank: int = 0, nranks: int = 1, device: int | None = None, stream=None,
                 nccl_id: bytes | None = None):
        import torch
        L = load()
        self._L = L
        self.cfg = cfg
        self.device = torch.cuda.current_device() if device is None else int(device)
        torch.cuda.set_device(self.device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self._id = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        self.dist = Dist(rank, nranks, self.device, C.cast(self._id, C.c_void_p) if self._id else None,
                         C.c_void_p(self.stream.cuda_stream))
        nb = C.c_size_t()
        self._check(L.hom2d_workspace_bytes(C.byref(cfg), C.byref(self.dist), C.byref(nb)), None)
        self.workspace = torch.empty(nb.value + 256, dtype=torch.uint8, device=f"cuda:{self.device}")
        base = self.workspace.data_ptr()
        aligned = (base + 255) & ~255
        h = C.c_void_p()
        self._check(L.hom2d_create(C.byref(cfg), C.byref(self.dist), C.c_void_p(aligned), nb.value, C.byref(h)),
                    None)
        self.h = h
        r0, nr, nv = C.c_int32(), C.c_int32(), C.c_int64()
        L.hom2d_local_extent(h, C.byref(r0), C.byref(nr), C.byref(nv))
        self.row0, self.nrows, self.n_values = r0.value, nr.value, nv.value

    # ---- error handling ----------------------------------------------------
    def _check(self, st, h="self"):
        if st:
            msg = ""
            if h == "self" and getattr(self, "h", None):
                msg = self._L.hom2d_last_error(self.h).decode(errors="replace")
            if st == 4:
                raise NonPhysicalState(st, msg)
            raise Hom2dError(st, msg)

    # ---- ABI mirror ----------------------------------------------------------
    def set_state(self, q, t0: float = 0.0):
        import torch
        if isinstance(q, torch.Tensor):
            assert q.dtype == torch.float64 and q.is_contiguous() and q.numel() == self.n_values
            on_dev = int(q.is_cuda)
            ptr = q.data_ptr()
        else:
            q = np.ascontiguousarray(q, dtype=np.float64)
            assert q.size == self.n_values
            on_dev, ptr = 0, q.ctypes.data
        self._check(self._L.hom2d_set_state(self.h, C.c_void_p(ptr), self.n_values, on_dev, float(t0)))

    def get_state(self, out=None):
        import torch
        if out is None:
            out = np.empty(self.n_values, dtype=np.float64)
        if isinstance(out, torch.Tensor):
            assert out.dtype == torch.float64 and out.is_contiguous() and out.numel() == self.n_values
            self._check(self._L.hom2d_get_state(self.h, C.c_void_p(out.data_ptr()), self.n_values, int(out.is_cuda)))
        else:
            self._check(self._L.hom2d_get_state(self.h, C.c_void_p(out.ctypes.data), self.n_values, 0))
        return out

    def init_case(self, case_id: int = VORTEX):
        self._check(self._L.hom2d_init_case(self.h, int(case_id)))

    def residual(self, q):
        """R(q) for a device tensor q (local strip); returns a new device tensor."""
        import torch
        assert q.is_cuda and q.dtype == torch.float64 and q.is_contiguous() and q.numel() == self.n_values
        r = torch.empty_like(q)
        self._check(self._L.hom2d_residual(self.h, C.c_void_p(q.data_ptr()), C.c_void_p(r.data_ptr())))
        return r

    def residual_strip(self, q, ghost_lo=None, ghost_hi=None):
        """R(q) of the local strip with explicit neighbour rows (device tensors)."""
        import torch
        assert q.is_cuda and q.dtype == torch.float64 and q.is_contiguous() and q.numel() == self.n_values
        r = torch.empty_like(q)
        ptr = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
        self._check(self._L.hom2d_residual_strip(self.h, ptr(q), ptr(ghost_lo), ptr(ghost_hi), ptr(r)))
        return r

    def limit(self):
        self._check(self._L.hom2d_limit(self.h))

    def compute_dt(self) -> float:
        dt = C.c_double()
        self._check(self._L.hom2d_compute_dt(self.h, C.byref(dt)))
        return dt.value

    def step(self, max_steps: int, t_end: float = math.inf):
        t, s = C.c_double(), C.c_int64()
        self._check(self._L.hom2d_step(self.h, int(max_steps), float(t_end), C.byref(t), C.byref(s)))
        return t.value, s.value

    def error(self, case_id: int = VORTEX, var: int = 0):
        l1, l2, li = C.c_double(), C.c_double(), C.c_double()
        self._check(self._L.hom2d_error(self.h, int(case_id), int(var), C.byref(l1), C.byref(l2), C.byref(li)))
        return l1.value, l2.value, li.value

    def time(self) -> float:
        t = C.c_double()
        self._check(self._L.hom2d_time(self.h, C.byref(t)))
        return t.value

    def decisions(self):
        out = np.zeros(8, dtype=np.int64)
        self._check(self._L.hom2d_decisions(self.h, C.c_void_p(out.ctypes.data)))
        return out

    def decision_map(self):
        """Per-element decision map (int64 [nx * nrows]); see hom2d_decision_map."""
        n = self.cfg.nx * self.nrows
        out = np.zeros(n, dtype=np.int64)
        self._check(self._L.hom2d_decision_map(self.h, C.c_void_p(out.ctypes.data), n))
        return out

    def launch_count(self) -> int:
        return int(self._L.hom2d_launch_count(self.h))

    def stage_timing(self, max_launches: int):
        self._check(self._L.hom2d_stage_timing(self.h, int(max_launches)))

    def stage_time(self):
        """(summed ms, number of timed stage-kernel launches) since the last call."""
        ms, n = C.c_double(), C.c_int64()
        self._check(self._L.hom2d_stage_time(self.h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def peer_id(self) -> bytes:
        """This rank's peer-memory halo id (hom2d_peer_id): plain bytes to exchange."""
        out = PeerId()
        self._check(self._L.hom2d_peer_id(self.h, C.byref(out)))
        return bytes(out)

    def peer_connect(self, lo: bytes, hi: bytes):
        """Map the strip neighbours' workspaces (hom2d_peer_connect): halos by peer memory from now on."""
        a, b = PeerId.from_buffer_copy(lo), PeerId.from_buffer_copy(hi)
        self._check(self._L.hom2d_peer_connect(self.h, C.byref(a), C.byref(b)))

    def close(self):
        if getattr(self, "h", None):
            grp = getattr(self, "_peer_group", False)
            if grp is not False:
                # peer-memory halo: a neighbour may still be pulling rows of this
                # workspace until every rank has returned from its last step
                import torch.distributed as dist
                if dist.is_initialized():
                    dist.barrier(group=grp)
                self._peer_group = False
            self._L.hom2d_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self._peer_group = False  # (no collective from a finaliser)
            self.close()
        except Exception:
            pass


def peer_neighbours(rank: int, nranks: int):
    """Ranks whose workspaces a rank maps for the peer-memory halo: its strip
    neighbours (hom2d_strip_plan peer_lo, peer_hi; periodic in y)."""
    return (rank + nranks - 1) % nranks, (rank + 1) % nranks


def connect_peers(solver: "Solver", group=None):
    """Peer-memory halo for a multi-rank solver: all-gather the ids over
    torch.distributed (host bytes), connect to the strip neighbours.  Argument
    marshalling only; the exchange itself runs in the library's kernels."""
    import torch.distributed as dist
    ids = [None] * dist.get_world_size(group)
    dist.all_gather_object(ids, solver.peer_id(), group=group)
    lo, hi = peer_neighbours(dist.get_rank(group), len(ids))
    solver.peer_connect(ids[lo], ids[hi])
    solver._peer_group = group  # close() then waits for every rank before the workspace goes
    return ids
