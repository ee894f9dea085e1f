"""B200-native nodal-DG Euler RHS + explicit RK stage (arXiv:1710.03887, Appendix A).

Thin ctypes binding of ``libdg_b200.so`` (C ABI in include/dg.h): the
functions below carry the C names and only marshal arguments -- every step
of the hot path runs in the library's sm_100a kernels.  PyTorch is used for
device memory (the bound workspace) and CUDA streams only.  There is no CPU
fallback: importing this package fails loudly if the library is missing.

``Solver`` is a small convenience owner of a ctx + its workspace tensor.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libdg_b200.so")

DG_OK, DG_EARG, DG_EMESH, DG_EBLOWUP, DG_ECUDA, DG_ENCCL, DG_EUNSUPPORTED, DG_ESTATE = 0, 2, 3, 4, 5, 6, 7, 8
DG_BC_INTERIOR, DG_BC_WALL, DG_BC_PASSTHROUGH, DG_BC_INFLOW = 0, 1, 2, 3
DG_RK_LSERK4, DG_RK_HEUN = 0, 1
DG_SCHEME_NODAL, DG_SCHEME_MODAL = 0, 1
DG_MAX_ORDER = 6
DG_MAX_SENSORS = 256

SYMBOLS = (
    "dg_mesh_create", "dg_destroy", "dg_last_error", "dg_sizes", "dg_workspace_bytes", "dg_bind_workspace",
    "dg_memory_report", "dg_get_nodes", "dg_set_state", "dg_get_state", "dg_get_time", "dg_rhs", "dg_rk_step",
    "dg_check", "dg_stable_dt", "dg_nccl_get_unique_id", "dg_comm_init", "dg_halo_info", "dg_halo_peer",
    "dg_halo_buffers", "dg_halo_records", "dg_stage_pack", "dg_stage_compute", "dg_stage_finish", "dg_rhs_compute",
    "dg_get_operators", "dg_get_maps", "dg_get_geometry", "dg_launch_count",
    "dg_sensors_set", "dg_sensors_sample", "dg_sensors_record", "dg_sensors_recorded",
    "dg_set_max_ctas", "dg_build_info", "dg_halo_exchange", "dg_set_nccl_ctas",
    "dg_spectrum",
)


class DGError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"dg status {status}: {msg}")
        self.status = status


class dg_mesh_desc(C.Structure):
    _fields_ = [
        ("order", C.c_int),
        ("nv", C.c_int64),
        ("vxyz", C.POINTER(C.c_double)),
        ("k", C.c_int64),
        ("etov", C.POINTER(C.c_int64)),
        ("etoe", C.POINTER(C.c_int64)),
        ("etof", C.POINTER(C.c_int8)),
        ("bc", C.POINTER(C.c_int8)),
        ("gamma", C.c_double),
        ("q_inf", C.c_double * 5),
        ("part", C.POINTER(C.c_int32)),
        ("nparts", C.c_int),
        ("lambda_mode", C.c_int),
        ("check_every", C.c_int),
        ("rk_scheme", C.c_int),
        ("inflow_alpha", C.c_double),
        ("scheme", C.c_int),
        ("inflow_time_scale", C.c_double),
        ("inflow_half_amplitude", C.c_double),
    ]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1710_03887_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, I, I64, D, S = C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_size_t
    pd, pi64, pi32 = C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int32)
    sig = {
        "dg_mesh_create": (I, [C.POINTER(dg_mesh_desc), I, C.POINTER(P)]),
        "dg_destroy": (None, [P]),
        "dg_last_error": (C.c_char_p, [P]),
        "dg_sizes": (I, [P, pi64, C.POINTER(I), C.POINTER(I)]),
        "dg_workspace_bytes": (S, [P]),
        "dg_bind_workspace": (I, [P, P, S, P]),
        "dg_memory_report": (I, [P, C.POINTER(S)]),
        "dg_get_nodes": (I, [P, pd, pd, pd]),
        "dg_set_state": (I, [P, P, P, P, P, P, I, D, P]),
        "dg_get_state": (I, [P, P, P, P, P, P, I, P]),
        "dg_get_time": (I, [P, pd]),
        "dg_rhs": (I, [P, D, P, P]),
        "dg_rk_step": (I, [P, D, I, P]),
        "dg_check": (I, [P, P]),
        "dg_stable_dt": (I, [P, D, pd, P]),
        "dg_nccl_get_unique_id": (I, [P]),
        "dg_comm_init": (I, [P, P, I]),
        "dg_halo_info": (I, [P, C.POINTER(I), pi64, pi64]),
        "dg_halo_peer": (I, [P, I, C.POINTER(I), pi64, pi64, pi64, pi64]),
        "dg_halo_buffers": (I, [P, C.POINTER(P), C.POINTER(P)]),
        "dg_halo_records": (I, [P, pi64, C.POINTER(C.c_int8), pi64, C.POINTER(C.c_int8)]),
        "dg_stage_pack": (I, [P, P]),
        "dg_stage_compute": (I, [P, I, D, I, P]),
        "dg_stage_finish": (I, [P, I, D]),
        "dg_rhs_compute": (I, [P, D, P, I, P]),
        "dg_get_operators": (I, [P, pd, pd, pd, pd, pd, pd, pd, pi32]),
        "dg_get_maps": (I, [P, pi64, pi64]),
        "dg_get_geometry": (I, [P, pd, pd, pd, pd]),
        "dg_launch_count": (I64, [P]),
        "dg_sensors_set": (I, [P, I, pd, pi32, P]),
        "dg_sensors_sample": (I, [P, P, I, P]),
        "dg_sensors_record": (I, [P, P, I64]),
        "dg_sensors_recorded": (I64, [P]),
        "dg_set_max_ctas": (I, [P, I]),
        "dg_set_nccl_ctas": (I, [P, I]),
        "dg_spectrum": (I, [P, C.c_int64, C.c_int64, P, P, P]),
        "dg_build_info": (C.c_char_p, []),
        "dg_halo_exchange": (I, [P, P]),
    }
    for name, (res, args) in sig.items():
        if not hasattr(lib, name):   # an older build: the call fails (AttributeError) when used
            continue
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


class _LazyLib:
    """The shared library, loaded on first use (so `python -m paper_1710_03887_b200.build`
    works on a fresh checkout); any use without the built library raises ImportError."""

    _handle = None

    def __getattr__(self, name):
        if _LazyLib._handle is None:
            _LazyLib._handle = _load()
        return getattr(_LazyLib._handle, name)


_lib = _LazyLib()


def load():
    """Load libdg_b200.so now (raises ImportError if it has not been built)."""
    return _lib.dg_last_error


def _ptr(a, ctype):
    return None if a is None else a.ctypes.data_as(C.POINTER(ctype))


def _check(status, ctx=None):
    if status != DG_OK:
        msg = _lib.dg_last_error(ctx)
        raise DGError(status, msg.decode() if msg else "")


# ---------------------------------------------------------------- C-named wrappers
def dg_mesh_create(order, vxyz, etov, bc, *, etoe=None, etof=None, gamma=1.4, q_inf=(1.4, 0, 0, 0, 2.5),
                   part=None, nparts=1, rank=0, lambda_mode=0, check_every=0, rk_scheme=DG_RK_LSERK4,
                   inflow_alpha=565.0, scheme=DG_SCHEME_NODAL, inflow_time_scale=0.0, inflow_half_amplitude=0.0):
    """Returns an opaque ctx handle (int).  Host arrays are copied by the library."""
    vxyz = np.ascontiguousarray(vxyz, dtype=np.float64)
    etov = np.ascontiguousarray(etov, dtype=np.int64)
    bc = np.ascontiguousarray(bc, dtype=np.int8)
    etoe = None if etoe is None else np.ascontiguousarray(etoe, dtype=np.int64)
    etof = None if etof is None else np.ascontiguousarray(etof, dtype=np.int8)
    part = None if part is None else np.ascontiguousarray(part, dtype=np.int32)
    d = dg_mesh_desc()
    d.order = int(order)
    d.nv = vxyz.shape[0]
    d.vxyz = _ptr(vxyz, C.c_double)
    d.k = etov.shape[0]
    d.etov = _ptr(etov, C.c_int64)
    d.etoe = _ptr(etoe, C.c_int64)
    d.etof = _ptr(etof, C.c_int8)
    d.bc = _ptr(bc, C.c_int8)
    d.gamma = float(gamma)
    for i in range(5):
        d.q_inf[i] = float(q_inf[i])
    d.part = _ptr(part, C.c_int32)
    d.nparts = int(nparts) if part is not None else 1
    d.lambda_mode = int(lambda_mode)
    d.check_every = int(check_every)
    d.rk_scheme = int(rk_scheme)
    d.inflow_alpha = float(inflow_alpha)
    d.scheme = int(scheme)
    d.inflow_time_scale = float(inflow_time_scale)
    d.inflow_half_amplitude = float(inflow_half_amplitude)
    out = C.c_void_p()
    _check(_lib.dg_mesh_create(C.byref(d), int(rank), C.byref(out)))
    return out.value


def dg_destroy(ctx):
    _lib.dg_destroy(ctx)


def dg_last_error(ctx=None) -> str:
    m = _lib.dg_last_error(ctx)
    return m.decode() if m else ""


def dg_sizes(ctx):
    k, np_, nfp = C.c_int64(), C.c_int(), C.c_int()
    _check(_lib.dg_sizes(ctx, C.byref(k), C.byref(np_), C.byref(nfp)), ctx)
    return k.value, np_.value, nfp.value


def dg_workspace_bytes(ctx) -> int:
    return int(_lib.dg_workspace_bytes(ctx))


def dg_bind_workspace(ctx, dptr: int, nbytes: int, stream: int):
    _check(_lib.dg_bind_workspace(ctx, dptr, nbytes, stream), ctx)


def dg_memory_report(ctx):
    b = (C.c_size_t * 7)()
    _check(_lib.dg_memory_report(ctx, b), ctx)
    return dict(zip(("state", "residual", "staging", "geometry", "connectivity", "operators", "halo"), list(b)))


def dg_get_nodes(ctx):
    k, np_, _ = dg_sizes(ctx)
    x, y, z = (np.empty(k * np_) for _ in range(3))
    _check(_lib.dg_get_nodes(ctx, _ptr(x, C.c_double), _ptr(y, C.c_double), _ptr(z, C.c_double)), ctx)
    return np.stack([x, y, z]).reshape(3, k, np_)


def dg_set_state(ctx, ptrs, on_device: bool, t: float, stream: int):
    _check(_lib.dg_set_state(ctx, *ptrs, int(on_device), float(t), stream), ctx)


def dg_get_state(ctx, ptrs, on_device: bool, stream: int):
    _check(_lib.dg_get_state(ctx, *ptrs, int(on_device), stream), ctx)


def dg_get_time(ctx) -> float:
    t = C.c_double()
    _check(_lib.dg_get_time(ctx, C.byref(t)), ctx)
    return t.value


def dg_rhs(ctx, t: float, out_ptr: int, stream: int):
    _check(_lib.dg_rhs(ctx, float(t), out_ptr, stream), ctx)


def dg_rk_step(ctx, dt: float, nsteps: int, stream: int):
    _check(_lib.dg_rk_step(ctx, float(dt), int(nsteps), stream), ctx)


def dg_set_max_ctas(ctx, max_ctas: int):
    _check(_lib.dg_set_max_ctas(ctx, int(max_ctas)), ctx)


def dg_set_nccl_ctas(ctx, nctas: int):
    _check(_lib.dg_set_nccl_ctas(ctx, int(nctas)), ctx)


def dg_spectrum(x_ptr: int, n: int, m: int, amp_ptr: int, db_ptr: int, stream: int):
    _check(_lib.dg_spectrum(x_ptr, int(n), int(m), amp_ptr, db_ptr, stream), None)


def dg_build_info() -> str:
    return _lib.dg_build_info().decode()


def dg_check(ctx, stream: int):
    _check(_lib.dg_check(ctx, stream), ctx)


def dg_stable_dt(ctx, cfl: float, stream: int) -> float:
    dt = C.c_double()
    _check(_lib.dg_stable_dt(ctx, float(cfl), C.byref(dt), stream), ctx)
    return dt.value


def dg_nccl_get_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(_lib.dg_nccl_get_unique_id(buf))
    return bytes(buf)


def dg_comm_init(ctx, uid: bytes, nranks: int):
    buf = (C.c_char * 128).from_buffer_copy(uid)
    _check(_lib.dg_comm_init(ctx, buf, int(nranks)), ctx)


def dg_halo_info(ctx):
    n, s, r = C.c_int(), C.c_int64(), C.c_int64()
    _check(_lib.dg_halo_info(ctx, C.byref(n), C.byref(s), C.byref(r)), ctx)
    return n.value, s.value, r.value


def dg_halo_peer(ctx, p: int):
    vals = [C.c_int()] + [C.c_int64() for _ in range(4)]
    _check(_lib.dg_halo_peer(ctx, p, *[C.byref(v) for v in vals]), ctx)
    return dict(zip(("rank", "send_off", "nsend", "recv_off", "nrecv"), [v.value for v in vals]))


def dg_halo_buffers(ctx):
    s, r = C.c_void_p(), C.c_void_p()
    _check(_lib.dg_halo_buffers(ctx, C.byref(s), C.byref(r)), ctx)
    return s.value, r.value


def dg_halo_records(ctx):
    _, ns, nr = dg_halo_info(ctx)
    sg, sf = np.empty(ns, dtype=np.int64), np.empty(ns, dtype=np.int8)
    rg, rf = np.empty(nr, dtype=np.int64), np.empty(nr, dtype=np.int8)
    _check(_lib.dg_halo_records(ctx, _ptr(sg, C.c_int64), _ptr(sf, C.c_int8), _ptr(rg, C.c_int64),
                                _ptr(rf, C.c_int8)), ctx)
    return sg, sf, rg, rf


def dg_halo_exchange(ctx, stream: int):
    _check(_lib.dg_halo_exchange(ctx, stream), ctx)


def dg_stage_pack(ctx, stream: int):
    _check(_lib.dg_stage_pack(ctx, stream), ctx)


def dg_stage_compute(ctx, s: int, dt: float, which: int, stream: int):
    _check(_lib.dg_stage_compute(ctx, int(s), float(dt), int(which), stream), ctx)


def dg_stage_finish(ctx, s: int, dt: float):
    _check(_lib.dg_stage_finish(ctx, int(s), float(dt)), ctx)


def dg_rhs_compute(ctx, t: float, out_ptr: int, which: int, stream: int):
    _check(_lib.dg_rhs_compute(ctx, float(t), out_ptr, int(which), stream), ctx)


def dg_get_operators(ctx):
    k, Np, Nfp = dg_sizes(ctx)
    r, s, t = (np.empty(Np) for _ in range(3))
    Dr, Ds, Dt = (np.empty((Np, Np)) for _ in range(3))
    LIFT = np.empty((Np, 4 * Nfp))
    Fm = np.empty((4, Nfp), dtype=np.int32)
    _check(_lib.dg_get_operators(ctx, *[_ptr(a, C.c_double) for a in (r, s, t, Dr, Ds, Dt, LIFT)],
                                 _ptr(Fm, C.c_int32)), ctx)
    return dict(r=r, s=s, t=t, Dr=Dr, Ds=Ds, Dt=Dt, LIFT=LIFT, Fmask=Fm)


def dg_get_maps(ctx):
    k, Np, Nfp = dg_sizes(ctx)
    vM = np.empty((k, 4, Nfp), dtype=np.int64)
    vP = np.empty((k, 4, Nfp), dtype=np.int64)
    _check(_lib.dg_get_maps(ctx, _ptr(vM, C.c_int64), _ptr(vP, C.c_int64)), ctx)
    return vM, vP


def dg_get_geometry(ctx):
    k, _, _ = dg_sizes(ctx)
    J, rx, n, fs = np.empty(k), np.empty((k, 3, 3)), np.empty((k, 4, 3)), np.empty((k, 4))
    _check(_lib.dg_get_geometry(ctx, *[_ptr(a, C.c_double) for a in (J, rx, n, fs)]), ctx)
    return dict(J=J, rx=rx, nx=n, Fscale=fs)


def dg_launch_count(ctx) -> int:
    return int(_lib.dg_launch_count(ctx))


# ---------------------------------------------------------------- convenience owner
def dg_sensors_set(ctx, xyz, stream: int):
    """Locate n points (n x 3) in this rank's elements; returns the public element index per
    point (-1: not on this rank)."""
    xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
    el = np.empty(len(xyz), dtype=np.int32)
    _check(_lib.dg_sensors_set(ctx, len(xyz), _ptr(xyz, C.c_double), _ptr(el, C.c_int32), stream), ctx)
    return el


def dg_sensors_sample(ctx, out_ptr: int, on_device: bool, stream: int):
    _check(_lib.dg_sensors_sample(ctx, out_ptr, int(on_device), stream), ctx)


def dg_sensors_record(ctx, dbuf_ptr, capacity: int):
    _check(_lib.dg_sensors_record(ctx, dbuf_ptr, capacity), ctx)


def dg_sensors_recorded(ctx) -> int:
    return int(_lib.dg_sensors_recorded(ctx))


class Solver:
    """Owns one ctx and its device workspace (a torch uint8 tensor)."""

    def __init__(self, order, vxyz, etov, bc, *, device=None, **kw):
        import torch
        self.torch = torch
        self.ctx = dg_mesh_create(order, vxyz, etov, bc, **kw)
        self.K, self.Np, self.Nfp = dg_sizes(self.ctx)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        nbytes = dg_workspace_bytes(self.ctx)
        self.ws = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        base = self.ws.data_ptr()
        aligned = (base + 255) // 256 * 256
        dg_bind_workspace(self.ctx, aligned, nbytes, self.stream)

    @property
    def stream(self) -> int:
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def nodes(self):
        return dg_get_nodes(self.ctx)

    def set_state(self, Q, t: float = 0.0):
        """Q: (5, K, Np) float64, a numpy array (host) or a torch CUDA tensor."""
        torch = self.torch
        if isinstance(Q, torch.Tensor) and Q.is_cuda:
            Q = Q.contiguous()
            self._keep = Q
            ptrs = [Q[i].data_ptr() for i in range(5)]
            dg_set_state(self.ctx, ptrs, True, t, self.stream)
        else:
            Qh = torch.from_numpy(np.ascontiguousarray(Q, dtype=np.float64)).pin_memory()
            self._keep = Qh
            ptrs = [Qh[i].data_ptr() for i in range(5)]
            dg_set_state(self.ctx, ptrs, False, t, self.stream)
            torch.cuda.current_stream(self.device).synchronize()

    def get_state(self, device: bool = False):
        torch = self.torch
        if device:
            out = torch.empty((5, self.K, self.Np), dtype=torch.float64, device=self.device)
            dg_get_state(self.ctx, [out[i].data_ptr() for i in range(5)], True, self.stream)
            return out
        out = torch.empty((5, self.K, self.Np), dtype=torch.float64).pin_memory()
        dg_get_state(self.ctx, [out[i].data_ptr() for i in range(5)], False, self.stream)
        torch.cuda.current_stream(self.device).synchronize()
        return out.numpy().copy()

    def rhs(self, t: float = 0.0, device: bool = False):
        torch = self.torch
        out = torch.empty((5, self.K, self.Np), dtype=torch.float64, device=self.device)
        dg_rhs(self.ctx, t, out.data_ptr(), self.stream)
        if device:
            return out
        return out.cpu().numpy()

    def set_max_ctas(self, n: int):
        """Cap the stage-kernel grid (0 = one CTA per SM); results do not depend on it."""
        dg_set_max_ctas(self.ctx, n)

    def step(self, dt: float, nsteps: int = 1):
        dg_rk_step(self.ctx, dt, nsteps, self.stream)

    def stable_dt(self, cfl: float) -> float:
        return dg_stable_dt(self.ctx, cfl, self.stream)

    # ---- point sensors
    def set_sensors(self, xyz):
        """Place sensors at points xyz (n x 3); returns each point's public element (-1: none)."""
        self._nsens = len(np.asarray(xyz).reshape(-1, 3))
        self._rec = None
        return dg_sensors_set(self.ctx, xyz, self.stream)

    def sample_sensors(self):
        """(n, 6) array: rho, m_x, m_y, m_z, E, p at every sensor (NaN rows: not on this rank)."""
        out = np.empty((self._nsens, 6), dtype=np.float64)
        if self._nsens:
            dg_sensors_sample(self.ctx, out.ctypes.data, False, self.stream)
        return out

    def record_sensors(self, capacity: int):
        """Record one sample per RK step into a device buffer of `capacity` samples."""
        self._rec = self.torch.empty((capacity, self._nsens, 6), dtype=self.torch.float64, device=self.device)
        dg_sensors_record(self.ctx, self._rec.data_ptr(), capacity)

    def sensor_record(self):
        """(samples recorded so far, n, 6) array."""
        n = dg_sensors_recorded(self.ctx)
        self.torch.cuda.current_stream(self.device).synchronize()
        return self._rec[:n].cpu().numpy()

    @property
    def time(self) -> float:
        return dg_get_time(self.ctx)

    def close(self):
        if getattr(self, "ctx", None):
            dg_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
