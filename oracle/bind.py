"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU oracle.

Importable only from tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs (the checker side). Three backends:

* ``oracle``     — oracle/libtgs_oracle.so, our C restatement (tgs_oracle.c); always buildable.
* ``ref_native`` — oracle/_ref/libtgs_ref_native.so, the unmodified reference render/backward
  (/root/reference/proj/core/src/rasterizer.cpp) with glibc libm.
* ``ref_cr``     — the same reference objects linked with the correctly-rounded expf/sincosf
  interposer (cr_libm.c): the numerics contract the GPU kernels implement.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libtgs_oracle.so")
REF_DIR = os.path.join(HERE, "_ref")

PARAM_FIELDS = ("px", "py", "rot", "lsx", "lsy", "rop", "cr", "cg", "cb")
ALL_FIELDS = PARAM_FIELDS + ("depth",)
P = C.POINTER
f32p, f64p, u8p = P(C.c_float), P(C.c_double), P(C.c_uint8)
u32p, i32p, i64p, u64p = P(C.c_uint32), P(C.c_int32), P(C.c_int64), P(C.c_uint64)


def _ptr(a, ct):
    return a.ctypes.data_as(ct) if a is not None else C.cast(None, ct)


def build(force: bool = False) -> None:
    """Build oracle/libtgs_oracle.so (and oracle/_ref when /root/reference exists)."""
    targets = ["oracle"]
    if os.path.isdir("/root/reference/proj/core/src"):
        targets.append("ref")
    if force:
        subprocess.check_call(["make", "-C", HERE, "clean"])
    subprocess.check_call(["make", "-s", "-C", HERE] + targets)


@dataclass
class Scene:
    """A 2-D Gaussian scene in model (creation) order — the reference's GaussianModel
    (model.hpp:45-152) flattened to SoA numpy arrays."""

    px: np.ndarray
    py: np.ndarray
    rot: np.ndarray
    lsx: np.ndarray
    lsy: np.ndarray
    rop: np.ndarray
    cr: np.ndarray
    cg: np.ndarray
    cb: np.ndarray
    depth: np.ndarray
    id: np.ndarray
    pos_acc: np.ndarray = None
    col_acc: np.ndarray = None
    accum: np.ndarray = None
    visit: np.ndarray = None
    window: np.ndarray = None
    tau_v: np.ndarray = None
    next_id: int = 0

    @property
    def n(self) -> int:
        return int(self.px.shape[0])

    @staticmethod
    def empty(n: int, capacity: int | None = None) -> "Scene":
        cap = max(capacity or n, 1)
        kw = {f: np.zeros(cap, np.float32) for f in ALL_FIELDS}
        s = Scene(**kw, id=np.zeros(cap, np.uint64))
        s.pos_acc = np.zeros(cap, np.float32)
        s.col_acc = np.zeros(cap, np.float32)
        s.accum = np.zeros(cap, np.int32)
        s.visit = np.zeros(cap, np.int64)
        s.window = np.zeros(cap, np.int64)
        s.tau_v = np.full(cap, 5.0, np.float64)
        return s.truncated(n)

    def truncated(self, n: int) -> "Scene":
        kw = {}
        for k, v in self.__dict__.items():
            kw[k] = v[:n] if isinstance(v, np.ndarray) else v
        return Scene(**kw)

    def copy(self) -> "Scene":
        kw = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in self.__dict__.items()}
        return Scene(**kw)

    def ensure_stats(self) -> "Scene":
        n = self.n
        if self.pos_acc is None:
            self.pos_acc = np.zeros(n, np.float32)
            self.col_acc = np.zeros(n, np.float32)
            self.accum = np.zeros(n, np.int32)
            self.visit = np.zeros(n, np.int64)
            self.window = np.zeros(n, np.int64)
        if self.tau_v is None:
            self.tau_v = np.full(n, 5.0, np.float64)
        return self

    def astype(self, dt) -> "Scene":
        s = self.copy()
        for f in ALL_FIELDS:
            setattr(s, f, getattr(s, f).astype(dt))
        return s


class OrScene(C.Structure):
    _fields_ = [("n", C.c_int64)] + [(f, f32p) for f in ALL_FIELDS] + [
        ("id", u64p), ("pos_acc", f32p), ("col_acc", f32p), ("accum", i32p), ("visit", i64p),
        ("window", i64p), ("tau_v", f64p), ("next_id", C.c_uint64)]


class OrPrepared(C.Structure):
    _fields_ = [(f, f32p) for f in ("mx", "my", "i00", "i01", "i11", "alpha", "c0", "c1", "c2",
                                     "rx", "ry")] + [("orig", u32p)]


class OrScreen(C.Structure):
    _fields_ = [(f, f32p) for f in ("gmx", "gmy", "gs00", "gs01", "gs11", "galpha", "gc0", "gc1",
                                     "gc2", "maxw")] + [("touched", u8p)]


class OrPcg(C.Structure):
    _fields_ = [("state", C.c_uint64), ("inc", C.c_uint64)]


class OrAdamCfg(C.Structure):
    _fields_ = [("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("lr", C.c_float * 9), ("bc1", C.c_float), ("bc2", C.c_float),
                ("ls_lo", C.c_float), ("ls_hi", C.c_float), ("raw_cap", C.c_float)]


class OrDensifyCfg(C.Structure):
    _fields_ = [("tau_pos", C.c_float), ("tau_color", C.c_float),
                ("opacity_mask_floor", C.c_float), ("opacity_prune_floor", C.c_float),
                ("color_branch_prob", C.c_float), ("tau_v_init", C.c_double),
                ("child_raw_opacity", C.c_float)]


class OrBudget(C.Structure):
    _fields_ = [(f, C.c_double) for f in ("n_init", "m_final", "m_adaptive", "alpha",
                                           "alpha_base", "ema")] + [
        ("has_ema", C.c_int)] + [(f, C.c_int64) for f in (
            "warmup_steps", "window_size", "refit_interval", "ma_depth", "last_refit")] + [
        ("lambda_", C.c_double), ("log_len", C.c_int64), ("log_cap", C.c_int64),
        ("log_t", f64p), ("log_ema", f64p), ("fit_len", C.c_int64), ("fit_cap", C.c_int64),
        ("fits", f64p)]


def _c_scene(s: Scene, keep: list) -> OrScene:
    """Marshal a Scene (float32 arrays, contiguous) into the oracle struct."""
    cs = OrScene()
    cs.n = s.n
    for f in ALL_FIELDS:
        a = np.ascontiguousarray(getattr(s, f), np.float32)
        if a is not getattr(s, f):
            setattr(s, f, a)
        setattr(cs, f, _ptr(a, f32p))
    cs.id = _ptr(s.id, u64p)
    cs.pos_acc = _ptr(s.pos_acc, f32p)
    cs.col_acc = _ptr(s.col_acc, f32p)
    cs.accum = _ptr(s.accum, i32p)
    cs.visit = _ptr(s.visit, i64p)
    cs.window = _ptr(s.window, i64p)
    cs.tau_v = _ptr(s.tau_v, f64p)
    cs.next_id = s.next_id
    keep.append(s)
    return cs


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.or_pcg32_next.restype = C.c_uint32
        L.or_pcg32_uniform.restype = C.c_double
        L.or_l1_loss.restype = C.c_double
        L.or_loss.restype = C.c_double
        L.or_loss.argtypes = [f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, f32p, C.c_float, f32p]
        for fn in ("or_select_candidates", "or_cap_candidates", "or_spawn", "or_prune",
                   "or_densify_event", "or_budget_at"):
            getattr(L, fn).restype = C.c_int64
        L.or_budget_t_norm.restype = C.c_double
        L.or_budget_t_norm.argtypes = [C.c_int64, C.c_int64, C.c_int64]
        L.or_budget_at.argtypes = [P(OrBudget), C.c_double]
        L.or_budget_record_loss.argtypes = [P(OrBudget), C.c_int64, C.c_double]
        L.or_budget_update.argtypes = [P(OrBudget), C.c_int64]
        L.or_budget_init.argtypes = [P(OrBudget), C.c_double, C.c_double]
        L.or_adam_config.argtypes = [P(OrAdamCfg), C.c_int64, C.c_int64, C.c_double]
        L.or_densify_config.argtypes = [P(OrDensifyCfg), C.c_float]
        L.or_pcg32_init.argtypes = [P(OrPcg), C.c_uint64, C.c_uint64]
        L.or_pcg32_advance.argtypes = [P(OrPcg), C.c_uint64]
        L.or_synthetic_scene.argtypes = [C.c_uint64, C.c_int64, C.c_int, C.c_int, P(OrScene)]
        _LIB = L
    return _LIB


def set_math(cr: bool) -> None:
    lib().or_set_math(1 if cr else 0)


# ------------------------------------------------------------------ generators / rng
def synthetic_scene(seed: int, n: int, W: int, H: int) -> Scene:
    s = Scene.empty(n)
    keep: list = []
    cs = _c_scene(s, keep)
    lib().or_synthetic_scene(seed, n, W, H, C.byref(cs))
    s.next_id = n
    return s


class Pcg32:
    def __init__(self, seed=0x853C49E6748FEA9B, stream=1):
        self.c = OrPcg()
        lib().or_pcg32_init(C.byref(self.c), seed, stream)

    def next_u32(self) -> int:
        return lib().or_pcg32_next(C.byref(self.c))

    def uniform(self) -> float:
        return lib().or_pcg32_uniform(C.byref(self.c))

    def advance(self, delta: int) -> None:
        lib().or_pcg32_advance(C.byref(self.c), delta)

    @property
    def state(self):
        return (self.c.state, self.c.inc)

    def set_state(self, st) -> None:
        self.c.state, self.c.inc = int(st[0]), int(st[1])


# ------------------------------------------------------------------ render / backward
def active_count(p, ox, oy, W, H):
    cols = (W - ox - 1) // p + 1 if W > ox else 0
    rows = (H - oy - 1) // p + 1 if H > oy else 0
    return cols * rows


class OracleError(Exception):
    def __init__(self, code, msg=""):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


def _ref_lib(kind: str):
    path = os.path.join(REF_DIR, f"libtgs_ref_{kind}.so")
    if not os.path.exists(path):
        raise FileNotFoundError(path)
    L = C.CDLL(path)
    return L


_REF = {}


def ref_lib(kind: str):
    if kind not in _REF:
        _REF[kind] = _ref_lib(kind)
    return _REF[kind]


def ref_available() -> bool:
    return all(os.path.exists(os.path.join(REF_DIR, f"libtgs_ref_{k}.so"))
               for k in ("native", "cr"))


class RefScene(C.Structure):
    _fields_ = [("n", C.c_int64)] + [(f, C.c_void_p) for f in ALL_FIELDS] + [
        ("ids", u64p), ("next_id", C.c_uint64), ("tau_v", f64p)]


def _ref_scene(s: Scene, dt, keep: list) -> RefScene:
    rs = RefScene()
    rs.n = s.n
    for f in ALL_FIELDS:
        a = np.ascontiguousarray(getattr(s, f), dt)
        keep.append(a)
        setattr(rs, f, a.ctypes.data)
    ids = np.ascontiguousarray(s.id, np.uint64)
    keep.append(ids)
    rs.ids = _ptr(ids, u64p)
    rs.next_id = max(s.next_id, int(ids.max()) + 1 if s.n else 0)
    if s.tau_v is not None:
        tv = np.ascontiguousarray(s.tau_v, np.float64)
        keep.append(tv)
        rs.tau_v = _ptr(tv, f64p)
    else:
        rs.tau_v = C.cast(None, f64p)
    return rs


def render(s: Scene, p, ox, oy, W, H, bg=(0, 0, 0), lowpass_p=0, impl="oracle", threads=1,
           dtype=np.float32):
    """Returns (rgb[P,3], T[P], blend_ops, evals or None)."""
    Pn = active_count(p, ox, oy, W, H)
    rgb = np.zeros((Pn, 3), dtype)
    T = np.zeros(Pn, dtype)
    ops = C.c_uint64(0)
    keep: list = []
    if impl == "oracle":
        ev = C.c_uint64(0)
        bgv = np.asarray(bg, np.float32)
        rc = lib().or_render(C.byref(_c_scene(s, keep)), p, ox, oy, W, H, _ptr(bgv, f32p),
                             lowpass_p, _ptr(rgb, f32p), _ptr(T, f32p), C.byref(ops), C.byref(ev))
        if rc:
            raise OracleError(rc)
        return rgb, T, ops.value, ev.value
    L = ref_lib(impl.split("_", 1)[1])
    err = C.create_string_buffer(256)
    rs = _ref_scene(s, dtype, keep)
    bgv = np.asarray(bg, dtype)
    fn = L.ref_render_f32 if dtype == np.float32 else L.ref_render_f64
    rc = fn(C.byref(rs), p, ox, oy, W, H, bgv.ctypes.data_as(C.c_void_p), threads, lowpass_p,
            rgb.ctypes.data_as(C.c_void_p), T.ctypes.data_as(C.c_void_p), C.byref(ops), err, 256)
    if rc:
        raise OracleError(rc, err.value.decode())
    return rgb, T, ops.value, None


def backward(s: Scene, p, ox, oy, W, H, dLdC, bg=(0, 0, 0), lowpass_p=0, impl="oracle",
             threads=1, update_stats=True, dtype=np.float32, screen=False):
    """Returns (grads[9, n], screen-space dict or None). Updates s's stats in place."""
    s.ensure_stats()
    n = s.n
    grads = np.zeros((9, max(n, 1)), dtype)
    keep: list = []
    dLdC = np.ascontiguousarray(dLdC, dtype)
    gp = (C.c_void_p * 9)(*[grads[q].ctypes.data for q in range(9)])
    scr = None
    if impl == "oracle":
        if dLdC.size // 3 != active_count(p, ox, oy, W, H):
            raise OracleError(1, "backward: loss-gradient count does not match pattern ranks")
        bgv = np.asarray(bg, np.float32)
        gpp = (f32p * 9)(*[_ptr(grads[q], f32p) for q in range(9)])
        sc = None
        if screen:
            scr = {k: np.zeros(max(n, 1), np.float32) for k in (
                "gmx", "gmy", "gs00", "gs01", "gs11", "galpha", "gc0", "gc1", "gc2", "maxw")}
            scr["touched"] = np.zeros(max(n, 1), np.uint8)
            sc = OrScreen(*[_ptr(scr[k], f32p) for k in (
                "gmx", "gmy", "gs00", "gs01", "gs11", "galpha", "gc0", "gc1", "gc2", "maxw")],
                _ptr(scr["touched"], u8p))
        rc = lib().or_backward(C.byref(_c_scene(s, keep)), p, ox, oy, W, H, _ptr(bgv, f32p),
                               _ptr(dLdC, f32p), lowpass_p, gpp,
                               C.byref(sc) if sc is not None else None, 1 if update_stats else 0)
        if rc:
            raise OracleError(rc)
        return grads[:, :n], scr
    L = ref_lib(impl.split("_", 1)[1])
    err = C.create_string_buffer(256)
    rs = _ref_scene(s, dtype, keep)
    bgv = np.asarray(bg, dtype)
    fn = L.ref_backward_f32 if dtype == np.float32 else L.ref_backward_f64
    st_dt = dtype
    pos = np.ascontiguousarray(s.pos_acc, st_dt)
    col = np.ascontiguousarray(s.col_acc, st_dt)
    acc = np.ascontiguousarray(s.accum, np.int32)
    vis = np.ascontiguousarray(s.visit, np.int64)
    win = np.ascontiguousarray(s.window, np.int64)
    rc = fn(C.byref(rs), p, ox, oy, W, H, bgv.ctypes.data_as(C.c_void_p),
            dLdC.ctypes.data_as(C.c_void_p), C.c_int64(dLdC.size // 3), threads, lowpass_p, gp,
            pos.ctypes.data_as(C.c_void_p), col.ctypes.data_as(C.c_void_p), _ptr(acc, i32p),
            _ptr(vis, i64p), _ptr(win, i64p), err, 256)
    if rc:
        raise OracleError(rc, err.value.decode())
    if update_stats:
        s.pos_acc[:] = pos.astype(np.float32) if dtype != np.float32 else pos
        s.col_acc[:] = col.astype(np.float32) if dtype != np.float32 else col
        s.accum[:] = acc
        s.visit[:] = vis
        s.window[:] = win
    return grads[:, :n], None


class RefSession:
    """One persistent tgs::GaussianModel<float> of the unmodified reference (oracle/_ref), kept
    across fit iterations so its cached blend order (model.hpp:105-119) is reused the way the
    reference's own trainer would reuse it; parameters are written in place between iterations.
    Used by bench.py's reference arm. The scene `s` stays the SoA source of truth for the
    restated optimizer (adam_step); push() copies its 9 parameters into the model."""

    def __init__(self, s: Scene, impl="ref_native"):
        self.h = None
        self.L = ref_lib(impl.split("_", 1)[1])
        L = self.L
        L.ref_session_create_f32.restype = C.c_void_p
        L.ref_session_create_f32.argtypes = [C.c_void_p, C.c_char_p, C.c_int]
        L.ref_session_destroy.argtypes = [C.c_void_p]
        L.ref_session_sort.argtypes = [C.c_void_p]
        L.ref_session_set_params_f32.argtypes = [C.c_void_p, C.c_void_p]
        L.ref_session_render_f32.argtypes = [C.c_void_p] + [C.c_int] * 5 + [
            C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_char_p, C.c_int]
        L.ref_session_backward_f32.argtypes = [C.c_void_p] + [C.c_int] * 5 + [
            C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_char_p, C.c_int]
        L.ref_session_visits.argtypes = [C.c_void_p, C.c_void_p]
        self.s = s
        keep: list = []
        err = C.create_string_buffer(256)
        self.h = L.ref_session_create_f32(C.byref(_ref_scene(s, np.float32, keep)), err, 256)
        if not self.h:
            raise OracleError(3, err.value.decode())

    def close(self):
        if self.h:
            self.L.ref_session_destroy(self.h)
            self.h = None

    __del__ = close

    def sort(self):
        self.L.ref_session_sort(self.h)

    def push(self):
        arrs = [np.ascontiguousarray(getattr(self.s, f), np.float32) for f in PARAM_FIELDS]
        ptrs = (C.c_void_p * 9)(*[a.ctypes.data for a in arrs])
        self.L.ref_session_set_params_f32(self.h, ptrs)

    def render(self, p, ox, oy, W, H, bg=(0, 0, 0), threads=1):
        Pn = active_count(p, ox, oy, W, H)
        rgb = np.zeros((Pn, 3), np.float32)
        T = np.zeros(Pn, np.float32)
        ops = C.c_uint64(0)
        bgv = np.asarray(bg, np.float32)
        err = C.create_string_buffer(256)
        rc = self.L.ref_session_render_f32(self.h, p, ox, oy, W, H, bgv.ctypes.data, threads,
                                           rgb.ctypes.data, T.ctypes.data, C.byref(ops), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return rgb, T, ops.value

    def backward(self, p, ox, oy, W, H, dLdC, bg=(0, 0, 0), threads=1):
        n = self.s.n
        grads = np.zeros((9, max(n, 1)), np.float32)
        gp = (C.c_void_p * 9)(*[grads[q].ctypes.data for q in range(9)])
        dLdC = np.ascontiguousarray(dLdC, np.float32)
        bgv = np.asarray(bg, np.float32)
        err = C.create_string_buffer(256)
        rc = self.L.ref_session_backward_f32(self.h, p, ox, oy, W, H, bgv.ctypes.data, dLdC.ctypes.data,
                                             C.c_int64(dLdC.size // 3), threads, gp, err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return grads[:, :n]

    def visits(self):
        out = np.zeros(max(self.s.n, 1), np.int64)
        self.L.ref_session_visits(self.h, out.ctypes.data)
        return out[:self.s.n]


PREP_FIELDS = ("mx", "my", "i00", "i01", "i11", "alpha", "c0", "c1", "c2", "rx", "ry")


def prepare(s: Scene, lowpass_p: int, impl="oracle"):
    """prepare_splats (rasterizer.cpp:23-46) -> dict of arrays in blend order (+ 'orig')."""
    n = s.n
    out = {k: np.zeros(max(n, 1), np.float32) for k in PREP_FIELDS}
    out["orig"] = np.zeros(max(n, 1), np.uint32)
    keep: list = []
    if impl == "oracle":
        op = OrPrepared(*[_ptr(out[k], f32p) for k in PREP_FIELDS], _ptr(out["orig"], u32p))
        rc = lib().or_prepare(C.byref(_c_scene(s, keep)), lowpass_p, C.byref(op))
        if rc:
            raise OracleError(rc)
    else:
        L = ref_lib(impl.split("_", 1)[1])
        err = C.create_string_buffer(256)
        arr = (f32p * 11)(*[_ptr(out[k], f32p) for k in PREP_FIELDS])
        rc = L.ref_prepare_f32(C.byref(_ref_scene(s, np.float32, keep)), lowpass_p, arr,
                               _ptr(out["orig"], u32p), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
    return {k: v[:n] for k, v in out.items()}


def tile_grid(s: Scene, lowpass_p: int, W: int, H: int, impl="oracle"):
    """build_tile_grid (rasterizer.cpp:67-102) -> (offsets[tiles+1], items[K])."""
    tiles = ((W + 15) // 16) * ((H + 15) // 16)
    offsets = np.zeros(tiles + 1, np.uint32)
    k = C.c_int64(0)
    keep: list = []
    if impl == "oracle":
        prep = prepare(s, lowpass_p)
        arrs = {kk: np.ascontiguousarray(v) for kk, v in prep.items()}
        keep.append(arrs)
        op = OrPrepared(*[_ptr(arrs[kk], f32p) for kk in PREP_FIELDS], _ptr(arrs["orig"], u32p))
        lib().or_tile_grid(C.byref(op), C.c_int64(s.n), W, H, _ptr(offsets, u32p), None,
                           C.c_int64(0), C.byref(k))
        items = np.zeros(max(k.value, 1), np.uint32)
        lib().or_tile_grid(C.byref(op), C.c_int64(s.n), W, H, _ptr(offsets, u32p),
                           _ptr(items, u32p), C.c_int64(k.value), C.byref(k))
        return offsets, items[:k.value]
    L = ref_lib(impl.split("_", 1)[1])
    err = C.create_string_buffer(256)
    rs = _ref_scene(s, np.float32, keep)
    L.ref_tile_grid_f32(C.byref(rs), lowpass_p, W, H, _ptr(offsets, u32p), None, C.c_int64(0),
                        C.byref(k), err, 256)
    items = np.zeros(max(k.value, 1), np.uint32)
    rc = L.ref_tile_grid_f32(C.byref(rs), lowpass_p, W, H, _ptr(offsets, u32p),
                             _ptr(items, u32p), C.c_int64(k.value), C.byref(k), err, 256)
    if rc:
        raise OracleError(rc, err.value.decode())
    return offsets, items[:k.value]


def sorted_order(s: Scene, impl="oracle"):
    out = np.zeros(max(s.n, 1), np.uint32)
    keep: list = []
    if impl == "oracle":
        lib().or_sorted_order(C.byref(_c_scene(s, keep)), _ptr(out, u32p))
    else:
        L = ref_lib(impl.split("_", 1)[1])
        err = C.create_string_buffer(256)
        L.ref_sorted_order_f32(C.byref(_ref_scene(s, np.float32, keep)), _ptr(out, u32p),
                               err, 256)
    return out[:s.n]


def knn(xy, k, impl="ref_native"):
    """k nearest neighbours of every point, self excluded, ascending (dist2, index).
    impl "ref_*": the reference KdTree2<float>::knn (kdtree.hpp:30-38, 96-116) per point;
    "brute": numpy restatement of the same ordering (float32 dist2, unfused)."""
    xy = np.ascontiguousarray(xy, np.float32).reshape(-1, 2)
    n = xy.shape[0]
    out = np.zeros((n, k), np.uint32)
    if impl == "brute":
        for i in range(n):
            dx = xy[i, 0] - xy[:, 0]
            dy = xy[i, 1] - xy[:, 1]
            d2 = (dx * dx).astype(np.float32) + (dy * dy).astype(np.float32)
            order = np.lexsort((np.arange(n), d2))
            order = order[order != i][:k]
            out[i, :len(order)] = order
            out[i, len(order):] = 0xFFFFFFFF
        return out
    L = ref_lib(impl.split("_", 1)[1])
    err = C.create_string_buffer(256)
    rc = L.ref_knn_f32(_ptr(xy, f32p), C.c_int64(n), int(k), _ptr(out, u32p), err, 256)
    if rc:
        raise OracleError(rc)
    return out


# ------------------------------------------------------------------ loss / adam / densify
def l1_loss(rgb, p, ox, oy, W, H, target):
    rgb = np.ascontiguousarray(rgb, np.float32)
    target = np.ascontiguousarray(target, np.float32)
    g = np.zeros_like(rgb)
    loss = lib().or_l1_loss(_ptr(rgb, f32p), p, ox, oy, W, H, _ptr(target, f32p), _ptr(g, f32p))
    return loss, g


def loss(rgb, p, ox, oy, W, H, target, ssim_weight=0.0):
    """compute_loss: dense (p = 1) (1-w) L1 + w (1 - SSIM), dilated L1 only.
    Returns (loss, dL/dC per active pixel)."""
    rgb = np.ascontiguousarray(rgb, np.float32)
    target = np.ascontiguousarray(target, np.float32)
    g = np.zeros_like(rgb)
    v = lib().or_loss(_ptr(rgb, f32p), p, ox, oy, W, H, _ptr(target, f32p), float(ssim_weight), _ptr(g, f32p))
    if v < 0:
        raise OracleError(1, "loss: bad pattern")
    return v, g


def adam_config(step, total_steps, diag) -> OrAdamCfg:
    c = OrAdamCfg()
    lib().or_adam_config(C.byref(c), step, total_steps, diag)
    return c


def adam_step(s: Scene, grads, m, v, cfg: OrAdamCfg):
    keep: list = []
    grads = np.ascontiguousarray(grads, np.float32)
    gp = (f32p * 9)(*[_ptr(grads[q], f32p) for q in range(9)])
    mp = (f32p * 9)(*[_ptr(m[q], f32p) for q in range(9)])
    vp = (f32p * 9)(*[_ptr(v[q], f32p) for q in range(9)])
    lib().or_adam_step(C.byref(_c_scene(s, keep)), gp, mp, vp, C.byref(cfg))


def densify_config(tau_pos=2e-4) -> OrDensifyCfg:
    c = OrDensifyCfg()
    lib().or_densify_config(C.byref(c), tau_pos)
    return c


def select_candidates(s: Scene, cfg, coin: bool):
    cand = np.zeros(max(s.n, 1), np.uint8)
    keep: list = []
    n = lib().or_select_candidates(C.byref(_c_scene(s, keep)), C.byref(cfg), 1 if coin else 0,
                                   _ptr(cand, u8p))
    return cand[:s.n], n


def cap_candidates(s: Scene, cand, budget_remaining):
    cand = np.ascontiguousarray(cand, np.uint8).copy()
    keep: list = []
    lib().or_cap_candidates(C.byref(_c_scene(s, keep)), _ptr(cand, u8p),
                            C.c_int64(budget_remaining))
    return cand


def densify_event(s: Scene, capacity: int, cfg, budget: int, rng: Pcg32, m=None, v=None):
    """One densify event (SPEC.md:575(3)). `s` (and the optional Adam moments m, v of shape
    [9, n]) are copied into capacity-sized arrays; returns (new_scene, spawned, pruned,
    candidates, (m, v)) with everything truncated to the new count."""
    s.ensure_stats()
    n0 = s.n
    cap = max(capacity, n0, 1)
    big = Scene.empty(cap, cap)
    for k, val in s.__dict__.items():
        if isinstance(val, np.ndarray):
            getattr(big, k)[:n0] = val
    big.next_id = s.next_id
    mm = vv = None
    if m is not None:
        mm = np.zeros((9, cap), np.float32)
        vv = np.zeros((9, cap), np.float32)
        mm[:, :n0] = m
        vv[:, :n0] = v
    keep: list = []
    cs = _c_scene(big, keep)
    cs.n = n0
    sp, pr, nc = C.c_int64(), C.c_int64(), C.c_int64()
    mp = (f32p * 9)(*[_ptr(mm[q], f32p) for q in range(9)]) if mm is not None else None
    vp = (f32p * 9)(*[_ptr(vv[q], f32p) for q in range(9)]) if vv is not None else None
    n = lib().or_densify_event(C.byref(cs), C.c_int64(cap), C.byref(cfg), C.c_int64(budget),
                               C.byref(rng.c), mp, vp, C.byref(sp), C.byref(pr), C.byref(nc))
    out = big.truncated(n)
    out.next_id = cs.next_id
    mv = (mm[:, :n].copy(), vv[:, :n].copy()) if mm is not None else None
    return out, sp.value, pr.value, nc.value, mv


def visit_audit(s: Scene):
    keep: list = []
    lib().or_visit_audit(C.byref(_c_scene(s, keep)))


class Budget:
    """BudgetController restated from SPEC.md:385-472 (oracle side)."""

    def __init__(self, n_init, m_final):
        self.c = OrBudget()
        lib().or_budget_init(C.byref(self.c), n_init, m_final)

    def __del__(self):
        try:
            lib().or_budget_free(C.byref(self.c))
        except Exception:
            pass

    def record_loss(self, t, loss):
        rc = lib().or_budget_record_loss(C.byref(self.c), t, loss)
        if rc:
            raise ValueError("loss must be > 0")

    def update(self, t):
        lib().or_budget_update(C.byref(self.c), t)

    def budget_at(self, t_norm):
        return lib().or_budget_at(C.byref(self.c), t_norm)

    @property
    def ema(self):
        return self.c.ema

    @property
    def alpha(self):
        return self.c.alpha

    @property
    def m_adaptive(self):
        return self.c.m_adaptive


def fit_power_exponent(t, y):
    t = np.ascontiguousarray(t, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    out = C.c_double()
    rc = lib().or_fit_power_exponent(_ptr(t, f64p), _ptr(y, f64p), C.c_int64(len(t)),
                                     C.byref(out))
    if rc:
        raise ValueError("insufficient data")
    return out.value


def budget_t_norm(step, warmup, densify_end):
    return lib().or_budget_t_norm(step, warmup, densify_end)


# ------------------------------------------------------------------ 3-D front end (ewa3d.c)
# parity unpinned at the reference (no 3-D code exists there); the
# restatement is pinned by formula KATs and FP64 finite differences (tests/test_oracle3d.py).
N3D = 59


class OrCamera(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("t", C.c_double * 3), ("fx", C.c_double),
                ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("znear", C.c_double), ("W", C.c_int), ("H", C.c_int)]


class OrAdam3dCfg(C.Structure):
    _fields_ = [(f, C.c_float) for f in ("beta1", "beta2", "eps", "lr_pos", "lr_rot", "lr_scale",
                                          "lr_opacity", "lr_dc", "lr_rest", "bc1", "bc2",
                                          "raw_cap")]


def camera_struct(cam) -> OrCamera:
    """`cam`: any object with R (3x3), t (3), fx, fy, cx, cy, znear, width, height."""
    c = OrCamera()
    R = np.asarray(cam.R, np.float64).reshape(9)
    for i in range(9):
        c.R[i] = float(R[i])
    for i in range(3):
        c.t[i] = float(cam.t[i])
    c.fx, c.fy, c.cx, c.cy, c.znear = (float(cam.fx), float(cam.fy), float(cam.cx),
                                       float(cam.cy), float(cam.znear))
    c.W, c.H = int(cam.width), int(cam.height)
    return c


def sh_basis(d):
    b = np.zeros(16, np.float64)
    db = np.zeros((16, 3), np.float64)
    lib().or3d_sh_basis(C.c_double(d[0]), C.c_double(d[1]), C.c_double(d[2]), _ptr(b, f64p),
                        _ptr(db, f64p))
    return b, db


def project3d(theta, cam, bump):
    """(status, out[12]) for one Gaussian in FP64: u v s00 s01 s11 alpha r g b depth rx ry."""
    th = np.ascontiguousarray(theta, np.float64)
    out = np.zeros(12, np.float64)
    cs = camera_struct(cam)
    rc = lib().or3d_project(_ptr(th, f64p), C.byref(cs), C.c_double(bump), _ptr(out, f64p))
    return rc, out


def chain3d(theta, cam, bump, screen):
    th = np.ascontiguousarray(theta, np.float64)
    sc = np.ascontiguousarray(screen, np.float64)
    g = np.zeros(N3D, np.float64)
    cs = camera_struct(cam)
    lib().or3d_chain(_ptr(th, f64p), C.byref(cs), C.c_double(bump), _ptr(sc, f64p), _ptr(g, f64p))
    return g


def _prep_arrays(n):
    nn = max(n, 1)
    arrs = {f: np.zeros(nn, np.float32) for f in ("mx", "my", "i00", "i01", "i11", "alpha", "c0",
                                                  "c1", "c2", "rx", "ry")}
    arrs["orig"] = np.zeros(nn, np.uint32)
    sp = OrPrepared(**{k: _ptr(v, f32p if v.dtype == np.float32 else u32p) for k, v in arrs.items()})
    return arrs, sp


def prepare3d(params, cam, lowpass_p):
    """Blend-ordered records of the visible Gaussians: dict of arrays (+ 'depth'), length nv."""
    params = np.ascontiguousarray(params, np.float32)
    n = params.shape[1]
    arrs, sp = _prep_arrays(n)
    depth = np.zeros(max(n, 1), np.float32)
    nv = C.c_int64(0)
    cs = camera_struct(cam)
    rc = lib().or3d_prepare(_ptr(params, f32p), C.c_int64(n), C.byref(cs), lowpass_p, C.byref(sp),
                            _ptr(depth, f32p), C.byref(nv))
    if rc:
        raise OracleError(rc)
    arrs["depth"] = depth
    return {k: v[:nv.value] for k, v in arrs.items()}


def render3d(params, cam, p, ox, oy, bg=(0, 0, 0), lowpass_p=0):
    params = np.ascontiguousarray(params, np.float32)
    n = params.shape[1]
    Pn = active_count(p, ox, oy, cam.width, cam.height)
    rgb = np.zeros((Pn, 3), np.float32)
    T = np.zeros(Pn, np.float32)
    ops, ev = C.c_uint64(0), C.c_uint64(0)
    bgv = np.asarray(bg, np.float32)
    cs = camera_struct(cam)
    rc = lib().or3d_render(_ptr(params, f32p), C.c_int64(n), C.byref(cs), p, ox, oy, _ptr(bgv, f32p),
                           lowpass_p, _ptr(rgb, f32p), _ptr(T, f32p), C.byref(ops), C.byref(ev))
    if rc:
        raise OracleError(rc)
    return rgb, T, ops.value, ev.value


def backward3d(params, cam, p, ox, oy, dLdC, bg=(0, 0, 0), lowpass_p=0):
    """(grads[59, n], screen[10, n], touched[n]) in row order."""
    params = np.ascontiguousarray(params, np.float32)
    n = params.shape[1]
    nn = max(n, 1)
    grads = np.zeros((N3D, nn), np.float32)
    scr = np.zeros((10, nn), np.float32)
    touched = np.zeros(nn, np.uint8)
    sg = OrScreen(*[_ptr(scr[q], f32p) for q in range(10)], _ptr(touched, u8p))
    dl = np.ascontiguousarray(dLdC, np.float32)
    bgv = np.asarray(bg, np.float32)
    cs = camera_struct(cam)
    rc = lib().or3d_backward(_ptr(params, f32p), C.c_int64(n), C.byref(cs), p, ox, oy,
                             _ptr(bgv, f32p), _ptr(dl, f32p), lowpass_p, _ptr(grads, f32p),
                             C.byref(sg))
    if rc:
        raise OracleError(rc)
    return grads[:, :n], scr[:, :n], touched[:n].astype(bool)


def adam3d_config(step, total_steps, extent) -> OrAdam3dCfg:
    c = OrAdam3dCfg()
    lib().or3d_adam_config(C.byref(c), C.c_int64(step), C.c_int64(total_steps), C.c_double(extent))
    return c


def adam3d_step(params, grads, m, v, cfg: OrAdam3dCfg):
    """In place on float32 [59, n] arrays."""
    n = params.shape[1]
    for a in (params, grads, m, v):
        assert a.dtype == np.float32 and a.flags.c_contiguous
    lib().or3d_adam_step(_ptr(params, f32p), _ptr(grads, f32p), _ptr(m, f32p), _ptr(v, f32p),
                         C.c_int64(n), C.byref(cfg))


# ------------------------------------------------------------------ 3-D densification (ewa3d.c)
class Or3dModel(C.Structure):
    _fields_ = [("n", C.c_int64), ("cap", C.c_int64), ("params", f32p), ("m1", f32p), ("m2", f32p),
                ("pos_acc", f32p), ("col_acc", f32p), ("visit", C.POINTER(C.c_int32)),
                ("visit_evt", C.POINTER(C.c_int32)), ("visit_aud", C.POINTER(C.c_int32)),
                ("id", C.POINTER(C.c_uint64)), ("tau_v", f64p), ("next_id", C.c_uint64)]


def densify3d_event(state: dict, cfg, budget: int, rng: Pcg32):
    """One 3-D densify event on `state` (dict of numpy arrays: params/m1/m2 [59][n], pos_acc,
    col_acc f32[n], visit, visit_evt, visit_aud i32[n], ids u64[n], tau_v f64[n], next_id) —
    or3d_densify_event, the restatement tgsx_densify3d is checked against. Returns the new state
    (length-n arrays) and (spawned, pruned, candidates, coin)."""
    n = state["params"].shape[1]
    cap = n + max(int(budget) - n, 0) + 1
    pad = lambda a, dt: np.concatenate([np.asarray(a, dt), np.zeros(cap - n, dt)])  # noqa: E731
    rows = lambda a: np.ascontiguousarray(  # noqa: E731
        np.concatenate([np.asarray(a, np.float32), np.zeros((N3D, cap - n), np.float32)], axis=1))
    P_, M1, M2 = rows(state["params"]), rows(state["m1"]), rows(state["m2"])
    pa, ca = pad(state["pos_acc"], np.float32), pad(state["col_acc"], np.float32)
    vi, ve, va = (pad(state[k], np.int32) for k in ("visit", "visit_evt", "visit_aud"))
    ids, tv = pad(state["ids"], np.uint64), pad(state["tau_v"], np.float64)
    I32 = C.POINTER(C.c_int32)
    m = Or3dModel(n, cap, _ptr(P_, f32p), _ptr(M1, f32p), _ptr(M2, f32p), _ptr(pa, f32p), _ptr(ca, f32p),
                  vi.ctypes.data_as(I32), ve.ctypes.data_as(I32), va.ctypes.data_as(I32),
                  ids.ctypes.data_as(C.POINTER(C.c_uint64)), _ptr(tv, f64p), int(state["next_id"]))
    sp, pr, nc = C.c_int64(), C.c_int64(), C.c_int64()
    coin = C.c_int()
    L = lib()
    L.or3d_densify_event.restype = C.c_int64
    L.or3d_densify_event.argtypes = [P(Or3dModel), P(OrDensifyCfg), C.c_int64, P(OrPcg), P(C.c_int64),
                                     P(C.c_int64), P(C.c_int64), P(C.c_int)]
    L.or3d_densify_event(C.byref(m), C.byref(cfg), int(budget), C.byref(rng.c), C.byref(sp), C.byref(pr),
                         C.byref(nc), C.byref(coin))
    k = m.n
    out = {"params": P_[:, :k].copy(), "m1": M1[:, :k].copy(), "m2": M2[:, :k].copy(), "pos_acc": pa[:k].copy(),
           "col_acc": ca[:k].copy(), "visit": vi[:k].copy(), "visit_evt": ve[:k].copy(),
           "visit_aud": va[:k].copy(), "ids": ids[:k].copy(), "tau_v": tv[:k].copy(), "next_id": m.next_id}
    return out, (sp.value, pr.value, nc.value, coin.value)


def visit_audit3d(state: dict):
    n = state["params"].shape[1]
    vi, va = np.ascontiguousarray(state["visit"], np.int32), np.ascontiguousarray(state["visit_aud"], np.int32).copy()
    tv = np.ascontiguousarray(state["tau_v"], np.float64).copy()
    I32 = C.POINTER(C.c_int32)
    dummy = np.zeros(1, np.float32)
    m = Or3dModel(n, n, _ptr(dummy, f32p), _ptr(dummy, f32p), _ptr(dummy, f32p), _ptr(dummy, f32p),
                  _ptr(dummy, f32p), vi.ctypes.data_as(I32), vi.ctypes.data_as(I32), va.ctypes.data_as(I32),
                  None, _ptr(tv, f64p), 0)
    lib().or3d_visit_audit(C.byref(m))
    return tv, va
