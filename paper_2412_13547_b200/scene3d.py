"""3-D front end of the fit hot path (BASELINE.json north_star item 1).

The reference is a 2-D analog of 3DGS with no camera or 3-D Gaussian: this module
adds the 3DGS front end in front of the same device binning / blend / backward as the 2-D path,
through the C ABI (include/tgsx.h, ``tgsx_*3d``):

* :class:`Camera` — pinhole camera, OpenCV axes, ``p_cam = R p + t``.
* :class:`GaussianModel3D` — host SoA parameters ``float32[59, n]``: mean xyz, quaternion wxyz,
  log-scales xyz, raw opacity, SH degree-3 coefficients ``sh[k][c]`` at row ``11 + 3k + c``.
* :class:`DeviceModel3D` — device-resident model: ``render``, ``backward``, ``adam_step``,
  ``fit_step`` (render -> L1 -> backward -> chain rule -> Adam, fused), ``stage_prepare``.

Same conventions as the 2-D API (api.py): patterns, low-pass bump, exceptions (``ValueError`` for
invalid input, ``RuntimeError`` for a degenerate covariance). No CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .api import Context, DilationPattern, RenderOptions, RenderOutput, default_context

N_PARAMS = 59
ROW_MEAN, ROW_QUAT, ROW_LOGSCALE, ROW_OPACITY, ROW_SH = 0, 3, 7, 10, 11
SH_C0 = 0.28209479177387814


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a):
    return C.c_void_p(a.ctypes.data) if a is not None else C.c_void_p(None)


@dataclass
class Camera:
    """Pinhole camera: u = fx x/z + cx, v = fy y/z + cy for p_cam = R p_world + t (x right,
    y down, z forward); pixel (i, j) has its centre at (i + 0.5, j + 0.5)."""

    R: np.ndarray
    t: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    znear: float = 0.2

    @staticmethod
    def look_at(eye, target, up, fov_x_deg: float, width: int, height: int, znear: float = 0.2):
        eye, target, up = (np.asarray(v, np.float64) for v in (eye, target, up))
        f = target - eye
        f /= np.linalg.norm(f)
        r = np.cross(f, up)
        r /= np.linalg.norm(r)
        d = np.cross(f, r)  # image y points down
        R = np.stack([r, d, f])
        fx = 0.5 * width / math.tan(math.radians(fov_x_deg) / 2)
        return Camera(R, -R @ eye, fx, fx, width / 2.0, height / 2.0, width, height, znear)

    @property
    def center(self):
        return -np.asarray(self.R, np.float64).T @ np.asarray(self.t, np.float64)

    def c(self) -> _lib.Camera3:
        c = _lib.Camera3()
        R = np.asarray(self.R, np.float64).reshape(9)
        for i in range(9):
            c.R[i] = float(R[i])
        for i in range(3):
            c.t[i] = float(self.t[i])
        c.fx, c.fy, c.cx, c.cy, c.znear = (float(self.fx), float(self.fy), float(self.cx),
                                           float(self.cy), float(self.znear))
        c.width, c.height = int(self.width), int(self.height)
        return c

    def pattern(self, p: int = 1, ox: int = 0, oy: int = 0) -> DilationPattern:
        return DilationPattern(p, ox, oy, self.width, self.height)


class GaussianModel3D:
    """Host parameters float32[59, n] (one row per component)."""

    def __init__(self, params: np.ndarray):
        params = _f32(params)
        if params.ndim != 2 or params.shape[0] != N_PARAMS:
            raise ValueError(f"params must be float32[{N_PARAMS}, n]")
        self.params = params

    def size(self) -> int:
        return int(self.params.shape[1])

    def __len__(self):
        return self.size()

    @staticmethod
    def synthetic(seed: int, n: int, cam: Camera, depth_range=(3.0, 6.0),
                  pixel_log_sigma=(0.0, 1.5), sh_rest: float = 0.1) -> "GaussianModel3D":
        """Seeded synthetic scene that covers the camera's image uniformly: pixel position
        U[0, W) x U[0, H), depth U[depth_range], per-axis scale = exp(U[pixel_log_sigma]) pixels
        at that depth (the 2-D generator's log-scale range), random rotation,
        raw opacity U[-2, 2), SH DC giving colours in ~[0.08, 0.92], higher bands U[-r, r)."""
        rng = np.random.default_rng(seed)
        u = rng.uniform(0, cam.width, n)
        v = rng.uniform(0, cam.height, n)
        z = rng.uniform(*depth_range, n)
        pc = np.stack([(u - cam.cx) * z / cam.fx, (v - cam.cy) * z / cam.fy, z])
        R = np.asarray(cam.R, np.float64)
        pw = R.T @ (pc - np.asarray(cam.t, np.float64)[:, None])
        P = np.zeros((N_PARAMS, n), np.float64)
        P[0:3] = pw
        q = rng.normal(size=(4, n))
        P[3:7] = q / np.linalg.norm(q, axis=0)
        P[7:10] = rng.uniform(*pixel_log_sigma, (3, n)) + np.log(z / cam.fx)[None]
        P[10] = rng.uniform(-2, 2, n)
        P[11:14] = rng.uniform(-1.5, 1.5, (3, n))
        P[14:] = rng.uniform(-sh_rest, sh_rest, (N_PARAMS - 14, n))
        return GaussianModel3D(P.astype(np.float32))


class DeviceModel3D:
    """Device-resident 3-D model (params, Adam moments, densify statistics) in HBM."""

    def __init__(self, ctx: Context | None = None, capacity: int = 1):
        self.ctx = ctx or default_context()
        h = C.c_void_p()
        self.ctx.check(self.ctx.L.tgsx_model3d_create(self.ctx.h, max(capacity, 1), C.byref(h)))
        self.h = h

    @staticmethod
    def from_host(model: GaussianModel3D, ctx: Context | None = None) -> "DeviceModel3D":
        d = DeviceModel3D(ctx, model.size())
        d.upload(model)
        return d

    def upload(self, model: GaussianModel3D):
        p = _f32(model.params)
        self.ctx.check(self.ctx.L.tgsx_model3d_upload(self.ctx.h, self.h, _ptr(p), p.shape[1]))

    def size(self) -> int:
        return int(self.ctx.L.tgsx_model3d_size(self.h))

    def download(self) -> GaussianModel3D:
        out = np.zeros((N_PARAMS, self.size()), np.float32)
        self.ctx.check(self.ctx.L.tgsx_model3d_download(self.ctx.h, self.h, _ptr(out), None, None, None))
        return GaussianModel3D(out)

    def stats(self):
        n = self.size()
        pos, col, vis = np.zeros(n, np.float32), np.zeros(n, np.float32), np.zeros(n, np.int32)
        self.ctx.check(self.ctx.L.tgsx_model3d_download(self.ctx.h, self.h, None, _ptr(pos),
                                                        _ptr(col), _ptr(vis)))
        return pos, col, vis

    def moments(self):
        n = self.size()
        m1, m2 = np.zeros((N_PARAMS, n), np.float32), np.zeros((N_PARAMS, n), np.float32)
        self.ctx.check(self.ctx.L.tgsx_model3d_download_moments(self.ctx.h, self.h, _ptr(m1), _ptr(m2)))
        return m1, m2

    def densify_state(self):
        """(ids u64[n], tau_v f64[n], visit count at the last densify event i32[n], at the last
        audit i32[n], next id) — tgsx_model3d_download_state."""
        n = self.size()
        ids, tau = np.zeros(n, np.uint64), np.zeros(n, np.float64)
        ve, va = np.zeros(n, np.int32), np.zeros(n, np.int32)
        nxt = C.c_uint64()
        self.ctx.check(self.ctx.L.tgsx_model3d_download_state(self.ctx.h, self.h, _ptr(ids), _ptr(tau), _ptr(ve),
                                                              _ptr(va), C.byref(nxt)))
        return ids, tau, ve, va, int(nxt.value)

    def densify(self, budget: int, rng_state: np.ndarray, config=None):
        """One densify event on the 3-D model (tgsx_densify3d: the SPEC's 2-D event on the 3-D
        parameters — select, top-k under the budget, spawn inside the parent's 1-sigma ellipsoid,
        prune, reset). rng_state (uint64[2], PCG32) is advanced in place."""
        from .api import densify_config
        cfg = config or densify_config()
        rep = _lib.DensifyReport()
        st = np.ascontiguousarray(rng_state, np.uint64)
        self.ctx.check(self.ctx.L.tgsx_densify3d(self.ctx.h, self.h, C.byref(cfg), int(budget),
                                                 st.ctypes.data_as(_lib.u64p), C.byref(rep)))
        rng_state[:] = st
        return rep

    def visit_audit(self):
        self.ctx.check(self.ctx.L.tgsx_visit_audit3d(self.ctx.h, self.h))

    def close(self):
        if getattr(self, "h", None):
            self.ctx.L.tgsx_model3d_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------ ops
    def render(self, cam: Camera, pattern: DilationPattern | None = None, background=(0.0, 0.0, 0.0),
               opts: RenderOptions | None = None) -> RenderOutput:
        opts = opts or RenderOptions()
        pattern = pattern or cam.pattern()
        P = pattern.active_count()
        rgb = np.zeros((P, 3), np.float32)
        T = np.zeros(P, np.float32)
        ops = C.c_uint64()
        bg = (C.c_float * 3)(*background)
        self.ctx.check(self.ctx.L.tgsx_render3d(self.ctx.h, self.h, C.byref(cam.c()), C.byref(pattern.c()),
                                                bg, opts.lowpass_p, _ptr(rgb), _ptr(T), C.byref(ops)))
        return RenderOutput(rgb, T, ops.value)

    def backward(self, cam: Camera, pattern: DilationPattern | None, background, pixel_loss_grads,
                 opts: RenderOptions | None = None, update_stats=True, screen=False):
        """Returns grads float32[59, n] (and the merged screen-space sums float32[10, n])."""
        opts = opts or RenderOptions()
        pattern = pattern or cam.pattern()
        g = _f32(pixel_loss_grads).reshape(-1, 3)
        n = self.size()
        out = np.zeros((N_PARAMS, n), np.float32)
        scr = np.zeros((10, n), np.float32) if screen else None
        bg = (C.c_float * 3)(*background)
        self.ctx.check(self.ctx.L.tgsx_backward3d(self.ctx.h, self.h, C.byref(cam.c()), C.byref(pattern.c()),
                                                  bg, opts.lowpass_p, _ptr(g), g.shape[0], _ptr(out),
                                                  _ptr(scr), 1 if update_stats else 0))
        return (out, scr) if screen else out

    def adam_step(self, grads, step: int, total_steps: int, scene_extent: float):
        g = _f32(grads)
        a = _lib.Adam3dArgs(step, total_steps, scene_extent)
        self.ctx.check(self.ctx.L.tgsx_adam3d_step(self.ctx.h, self.h, _ptr(g), C.byref(a)))

    def fit_step(self, cam: Camera, pattern: DilationPattern | None, background, target, step: int,
                 total_steps: int, scene_extent: float) -> float:
        """render -> L1 (+ SSIM on dense views when the context's weight is set) -> backward ->
        chain rule -> statistics -> Adam, fused. `target`: (H, W, 3) float32 host array or a
        device pointer (int)."""
        pattern = pattern or cam.pattern()
        a = _lib.Adam3dArgs(step, total_steps, scene_extent)
        bg = (C.c_float * 3)(*background)
        tp = C.c_void_p(target) if isinstance(target, int) else _ptr(_f32(target))
        loss = np.zeros(1, np.float32)
        self.ctx.check(self.ctx.L.tgsx_fit_step3d(self.ctx.h, self.h, C.byref(cam.c()), C.byref(pattern.c()),
                                                  bg, tp, C.byref(a), _ptr(loss)))
        return float(loss[0])

    def view_accumulate(self, cam: Camera, pattern: DilationPattern | None, background, target) -> float:
        """One view of a batched step: render -> L1 -> backward -> chain rule, summed into the step
        buffer (no parameter update)."""
        pattern = pattern or cam.pattern()
        bg = (C.c_float * 3)(*background)
        tp = C.c_void_p(target) if isinstance(target, int) else _ptr(_f32(target))
        loss = np.zeros(1, np.float32)
        self.ctx.check(self.ctx.L.tgsx_view_accumulate3d(self.ctx.h, self.h, C.byref(cam.c()),
                                                         C.byref(pattern.c()), bg, tp, _ptr(loss)))
        return float(loss[0])

    def step_buffer(self):
        """(device pointer, float count) of the [62][capacity] step buffer (for the all-reduce)."""
        n = C.c_int64()
        ptr = self.ctx.L.tgsx_step_buffer3d(self.h, C.byref(n))
        return int(ptr), int(n.value)

    def step_layout(self):
        """3-D rows stay in creation order on every rank: nothing to do (2-D API parity)."""

    def allreduce_step(self):
        """In-place sum of the packed [62][n] step buffer over the context's NCCL communicator."""
        self.ctx.check(self.ctx.L.tgsx_allreduce_step3d(self.ctx.h, self.h))

    def apply_step(self, batch_views: int, step: int, total_steps: int, scene_extent: float):
        a = _lib.Adam3dArgs(step, total_steps, scene_extent)
        self.ctx.check(self.ctx.L.tgsx_apply_step3d(self.ctx.h, self.h, batch_views, C.byref(a)))

    def stage_prepare(self, cam: Camera, lowpass_p: int = 1):
        """Blend-ordered records of the visible Gaussians: dict of arrays (mx, my, i00, i01, i11,
        alpha, c0, c1, c2, rx, ry, orig, depth)."""
        n = self.size()
        rec = np.zeros((max(n, 1), 16), np.float32)
        keys = np.zeros(max(n, 1), np.uint32)
        ordered = C.c_int32()
        self.ctx.check(self.ctx.L.tgsx_stage_prepare3d(self.ctx.h, self.h, C.byref(cam.c()), lowpass_p,
                                                       _ptr(rec), _ptr(keys), C.byref(ordered)))
        rec, keys = rec[:n], keys[:n]
        if not ordered.value:  # row order: the blend order is (depth key, row)
            rows = np.arange(n, dtype=np.uint64)
            order = np.argsort((keys.astype(np.uint64) << np.uint64(32)) | rows, kind="stable")
            rec, keys = rec[order], keys[order]
        nv = int(np.count_nonzero(keys != 0xFFFFFFFF))
        r = rec[:nv]  # Prepared: (mx, my, i00, i01) (i11, alpha, rx, ry) (r, g, b, orig) (rect)
        out = {"mx": r[:, 0], "my": r[:, 1], "i00": r[:, 2], "i01": r[:, 3], "i11": r[:, 4],
               "alpha": r[:, 5], "rx": r[:, 6], "ry": r[:, 7], "c0": r[:, 8], "c1": r[:, 9],
               "c2": r[:, 10], "orig": r[:, 11].view(np.uint32).copy(),
               "depth": (keys[:nv] & 0x7FFFFFFF).view(np.float32).copy(), "blend_ordered": bool(ordered.value)}
        return out


__all__ = ["Camera", "GaussianModel3D", "DeviceModel3D", "N_PARAMS", "SH_C0"]


class Trainer3D:
    """The SPEC fit loop (warm-up, densify every 20 with the convergence-aware budget, post-densify
    random dilation with SSIM on dense iterations, batched finale, visit audits) over a set of
    cameras of a DeviceModel3D (libtgsx tgsx_trainer3d_*, csrc/trainer.cpp)."""

    def __init__(self, dm: DeviceModel3D, cameras, scene_extent: float, config=None, **kw):
        from .api import train_config
        self.dm = dm
        self.cfg = config or train_config(**kw)
        self.cams = (_lib.Camera3 * len(cameras))(*[c.c() for c in cameras])
        h = C.c_void_p()
        dm.ctx.check(dm.ctx.L.tgsx_trainer3d_create(dm.ctx.h, dm.h, C.byref(self.cfg), self.cams, len(cameras),
                                                    float(scene_extent), C.byref(h)))
        self.h = h
        self._targets = None

    def set_targets(self, targets):
        """targets[v]: camera v's (H, W, 3) float32 host array or device pointer (int)."""
        self._keep = [t if isinstance(t, int) else _f32(t) for t in targets]
        ptrs = [t if isinstance(t, int) else t.ctypes.data for t in self._keep]
        self._targets = (C.c_void_p * len(ptrs))(*ptrs)

    def step(self) -> _lib.TrainReport:
        rep = _lib.TrainReport()
        self.dm.ctx.check(self.dm.ctx.L.tgsx_trainer3d_step(self.h, self._targets, len(self._targets),
                                                            C.byref(rep)))
        return rep

    def losses(self, max_n: int = 4096) -> np.ndarray:
        out = np.zeros(max_n, np.float32)
        n = C.c_int64()
        self.dm.ctx.check(self.dm.ctx.L.tgsx_trainer3d_losses(self.h, out.ctypes.data_as(_lib.f32p), max_n,
                                                              C.byref(n)))
        return out[:n.value]

    def close(self):
        if getattr(self, "h", None):
            self.dm.ctx.L.tgsx_trainer3d_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
