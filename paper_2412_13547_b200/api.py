"""Python mirror of the reference's hot-path interface, backed by libtgsx (CUDA, sm_100a).

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/core/include/tgs/*.hpp):

  GaussianModel   model.hpp:45-152 (+ DensifyStats model.hpp:17-40), host SoA numpy arrays
  DilationPattern dilation.hpp:14-56;  next_offsets dilation.hpp:60-64; lowpass_bump :67-70
  RenderOptions   rasterizer.hpp:48-53
  render          rasterizer.hpp:58-60  -> RenderOutput (rasterizer.hpp:21-26)
  backward        rasterizer.hpp:66-69  -> GradientSet (rasterizer.hpp:28-46), updates stats

plus the device-resident fast path the C ABI adds (DeviceModel, fit_step, batched views,
densify, BudgetController).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, load

PARAM_ROWS = ("px", "py", "rot", "lsx", "lsy", "rop", "cr", "cg", "cb", "depth")


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a, ct=C.c_void_p):
    if a is None:
        return None
    return a.ctypes.data_as(ct) if ct is not C.c_void_p else C.c_void_p(a.ctypes.data)


# ---------------------------------------------------------------- pattern
class DilationPattern:
    """Strided sampling pattern (dilation.hpp:14-56)."""

    def __init__(self, pattern_size: int, offset_x: int, offset_y: int, width: int, height: int):
        if pattern_size < 1:
            raise ValueError("dilation must be >= 1")
        if offset_x < 0 or offset_y < 0 or offset_x >= pattern_size or offset_y >= pattern_size:
            raise ValueError("dilation offsets must lie in [0, p)")
        if width < 1 or height < 1:
            raise ValueError("image dimensions must be >= 1")
        self.p, self.ox, self.oy, self.width, self.height = (
            pattern_size, offset_x, offset_y, width, height)
        self.cols = (width - offset_x - 1) // pattern_size + 1 if width > offset_x else 0
        self.rows = (height - offset_y - 1) // pattern_size + 1 if height > offset_y else 0

    def active(self, x, y):
        return x % self.p == self.ox and y % self.p == self.oy

    def active_count(self) -> int:
        return self.cols * self.rows

    def rank_of(self, x, y):
        return ((y - self.oy) // self.p) * self.cols + (x - self.ox) // self.p

    def pixel_at_rank(self, rank):
        return self.ox + (rank % self.cols) * self.p, self.oy + (rank // self.cols) * self.p

    def pattern_size(self):
        return self.p

    def active_pixels(self):
        """(x, y) integer arrays of the active pixels in rank order."""
        r = np.arange(self.active_count())
        return self.ox + (r % self.cols) * self.p, self.oy + (r // self.cols) * self.p

    def c(self) -> _lib.Pattern:
        return _lib.Pattern(self.p, self.ox, self.oy, self.width, self.height)


def next_offsets(p: int, iteration: int):
    """dilation.hpp:60-64"""
    if p < 1:
        raise ValueError("dilation must be >= 1")
    idx = iteration % (p * p)
    return idx % p, idx // p


def lowpass_bump(p: int) -> float:
    """dilation.hpp:67-70 (float arithmetic)"""
    return float(np.float32(0.3) + np.float32(0.5) * np.float32(p - 1))


@dataclass
class RenderOptions:
    threads: int = 1     # accepted for API parity; the GPU path ignores it
    lowpass_p: int = 0   # 0 => the pattern's p (rasterizer.cpp:138-140)


@dataclass
class RenderOutput:
    colors: np.ndarray               # (P, 3) by dense rank
    final_transmittance: np.ndarray  # (P,)
    blend_op_count: int = 0


@dataclass
class GradientSet:
    position: np.ndarray    # (n, 2)
    rotation: np.ndarray    # (n,)
    log_scales: np.ndarray  # (n, 2)
    raw_opacity: np.ndarray
    color: np.ndarray       # (n, 3)

    def size(self):
        return self.rotation.shape[0]

    @staticmethod
    def from_rows(g: np.ndarray) -> "GradientSet":
        return GradientSet(np.stack([g[0], g[1]], 1), g[2].copy(), np.stack([g[3], g[4]], 1),
                           g[5].copy(), np.stack([g[6], g[7], g[8]], 1))

    def rows(self) -> np.ndarray:
        return np.stack([self.position[:, 0], self.position[:, 1], self.rotation,
                         self.log_scales[:, 0], self.log_scales[:, 1], self.raw_opacity,
                         self.color[:, 0], self.color[:, 1], self.color[:, 2]]).astype(np.float32)


# ---------------------------------------------------------------- host model
class GaussianModel:
    """Host-side scene container with the reference's fields (model.hpp:45-152), stored as
    SoA float32 rows in model (creation) order."""

    def __init__(self, n: int = 0):
        self.params = np.zeros((10, n), np.float32)
        self.id = np.arange(n, dtype=np.uint64)
        self.pos_grad_norm_accum = np.zeros(n, np.float32)
        self.color_grad_norm_accum = np.zeros(n, np.float32)
        self.accum_count = np.zeros(n, np.int32)
        self.visit_count = np.zeros(n, np.int64)
        self.window_visit_count = np.zeros(n, np.int64)
        self.visit_thresholds = np.full(n, 5.0, np.float64)
        self._next_id = n

    # reference accessors
    def size(self):
        return self.params.shape[1]

    def __len__(self):
        return self.size()

    def next_id(self):
        return self._next_id

    def set_next_id(self, v):
        self._next_id = int(v)

    def row(self, name):
        return self.params[PARAM_ROWS.index(name)]

    def add(self, position, rotation, log_scales, raw_opacity, color, depth_key,
            visit_threshold=5.0) -> int:
        """GaussianModel::add (model.hpp:66-73): appends with the next creation id."""
        col = np.array([position[0], position[1], rotation, log_scales[0], log_scales[1],
                        raw_opacity, color[0], color[1], color[2], depth_key], np.float32)[:, None]
        self.params = np.concatenate([self.params, col], 1)
        gid = self._next_id
        self._next_id += 1
        self.id = np.append(self.id, np.uint64(gid))
        self.pos_grad_norm_accum = np.append(self.pos_grad_norm_accum, np.float32(0))
        self.color_grad_norm_accum = np.append(self.color_grad_norm_accum, np.float32(0))
        self.accum_count = np.append(self.accum_count, np.int32(0))
        self.visit_count = np.append(self.visit_count, np.int64(0))
        self.window_visit_count = np.append(self.window_visit_count, np.int64(0))
        self.visit_thresholds = np.append(self.visit_thresholds, visit_threshold)
        return gid

    def compact(self, keep) -> int:
        """GaussianModel::compact (model.hpp:77-103)."""
        keep = np.asarray(keep, bool)
        if keep.shape[0] != self.size():
            raise ValueError("keep mask size mismatch")
        removed = int((~keep).sum())
        self.params = np.ascontiguousarray(self.params[:, keep])
        for f in ("id", "pos_grad_norm_accum", "color_grad_norm_accum", "accum_count",
                  "visit_count", "window_visit_count", "visit_thresholds"):
            setattr(self, f, np.ascontiguousarray(getattr(self, f)[keep]))
        return removed

    @staticmethod
    def synthetic(seed: int, n: int, width: int, height: int) -> "GaussianModel":
        """Seeded synthetic scene generated by libtgsx's host generator."""
        m = GaussianModel(n)
        hs = m._host_scene()
        load().tgsx_synthetic_scene(seed, n, width, height, C.byref(hs))
        m._next_id = n
        return m

    def _host_scene(self) -> _lib.HostScene:
        self.params = np.ascontiguousarray(self.params, np.float32)
        hs = _lib.HostScene()
        hs.n = self.size()
        for i, f in enumerate(PARAM_ROWS):
            setattr(hs, f, self.params[i].ctypes.data_as(_lib.f32p))
        self.id = np.ascontiguousarray(self.id, np.uint64)
        hs.id = self.id.ctypes.data_as(_lib.u64p)
        hs.next_id = self._next_id
        for f, attr, ct in (("pos_acc", "pos_grad_norm_accum", _lib.f32p),
                            ("col_acc", "color_grad_norm_accum", _lib.f32p),
                            ("accum", "accum_count", _lib.i32p),
                            ("visit", "visit_count", _lib.i64p),
                            ("window", "window_visit_count", _lib.i64p),
                            ("tau_v", "visit_thresholds", _lib.f64p)):
            a = np.ascontiguousarray(getattr(self, attr))
            setattr(self, attr, a)
            setattr(hs, f, a.ctypes.data_as(ct))
        return hs

    def copy(self) -> "GaussianModel":
        m = GaussianModel(0)
        for k, v in self.__dict__.items():
            setattr(m, k, v.copy() if isinstance(v, np.ndarray) else v)
        return m


# ---------------------------------------------------------------- device objects
class Context:
    """A tgsx context: one CUDA stream + reusable workspace (one per host thread)."""

    def __init__(self, device: int = 0):
        self.L = load()
        h = C.c_void_p()
        rc = self.L.tgsx_create(device, C.byref(h))
        if rc:
            raise _lib.TgsxError(f"tgsx_create failed ({rc}): no usable CUDA device")
        self.h = h

    def close(self):
        if self.h:
            self.L.tgsx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc, what=""):
        check(rc, self.h, what)

    def synchronize(self):
        self.check(self.L.tgsx_synchronize(self.h))

    def set_stream(self, stream_handle: int):
        self.check(self.L.tgsx_set_stream(self.h, C.c_void_p(stream_handle)))

    @property
    def launches(self) -> int:
        return int(self.L.tgsx_launch_count(self.h))

    STAGES = ("depth_sort", "preprocess", "scan", "duplicate", "radix_sort", "ranges",
              "blend_forward", "blend_backward", "chain_adam", "loss", "densify", "adam")

    def profile(self, enable: bool = True):
        self.check(self.L.tgsx_profile(self.h, 1 if enable else 0))

    # ------------------------------------------------ in-library NCCL
    @staticmethod
    def _nccl_from_torch():
        """libtgsx dlopens "libnccl.so.2" on first use; inside a Python process that library must
        be PyTorch's own NCCL (torch's CUDA library needs its NCCL's symbols — a system NCCL loaded
        first would shadow it and break a later `import torch`). Importing torch loads it."""
        try:
            import torch  # noqa: F401
        except ImportError:
            pass

    @staticmethod
    def comm_unique_id() -> bytes:
        """A fresh 128-byte NCCL unique id (rank 0 creates it, the caller distributes it)."""
        Context._nccl_from_torch()
        buf = (C.c_uint8 * 128)()
        rc = _lib.load().tgsx_comm_unique_id(buf)
        if rc:
            raise RuntimeError(f"tgsx_comm_unique_id failed ({rc}): NCCL not loadable")
        return bytes(buf)

    def comm_init(self, unique_id: bytes, nranks: int, rank: int):
        """Attach an NCCL communicator of `nranks` (this context's device) for batched steps."""
        if len(unique_id) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        Context._nccl_from_torch()
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        self.check(self.L.tgsx_comm_init(self.h, buf, int(nranks), int(rank)))

    def comm_destroy(self):
        self.check(self.L.tgsx_comm_destroy(self.h))

    def comm_size(self) -> int:
        return int(self.L.tgsx_comm_size(self.h))

    def pipeline_timeline(self):
        """Per-bucket event times (ms from the step start) of the last profiled batched step:
        array [buckets][6] = chain start/end, all-reduce start/end, Adam start/end."""
        n = self.L.tgsx_pipeline_timeline(self.h, None, 0)
        out = np.zeros(max(n, 1), np.float32)
        self.L.tgsx_pipeline_timeline(self.h, _ptr(out, _lib.f32p), n)
        return out[:n].reshape(-1, 6)

    def set_binning(self, mode: int):
        """0: slab binning with per-tile sorts (default); 1: always the onesweep paths."""
        self.check(self.L.tgsx_set_binning(self.h, int(mode)))

    def set_ssim_weight(self, weight: float):
        """lambda_ssim of dense fused fit views (0 = L1 only)."""
        self.check(self.L.tgsx_set_ssim_weight(self.h, float(weight)))

    def profile_read(self):
        n = len(self.STAGES)
        ms = (C.c_double * n)()
        cnt = (C.c_int64 * n)()
        self.check(self.L.tgsx_profile_read(self.h, ms, cnt, n))
        return {s: (ms[i], cnt[i]) for i, s in enumerate(self.STAGES)}

    def graph_stats(self):
        """(captures, replayed launches, eager re-runs) of tgsx_fit_graph_step on this context."""
        c, r, e = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.check(self.L.tgsx_fit_graph_stats(self.h, C.byref(c), C.byref(r), C.byref(e)))
        return c.value, r.value, e.value

    def counters(self):
        ops, ev, pairs = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.check(self.L.tgsx_stage_counters(self.h, C.byref(ops), C.byref(ev), C.byref(pairs)))
        return {"blend_ops": ops.value, "evals": ev.value, "pairs": pairs.value}


_DEFAULT_CTX = None


def default_context() -> Context:
    global _DEFAULT_CTX
    if _DEFAULT_CTX is None:
        _DEFAULT_CTX = Context(0)
    return _DEFAULT_CTX


class DeviceModel:
    """Device-resident SoA model (params, ids, stats, tau_v, Adam moments) in HBM."""

    def __init__(self, ctx: Context | None = None, capacity: int = 1):
        self.ctx = ctx or default_context()
        h = C.c_void_p()
        self.ctx.check(self.ctx.L.tgsx_model_create(self.ctx.h, max(capacity, 1), C.byref(h)))
        self.h = h

    @staticmethod
    def from_host(model: GaussianModel, ctx: Context | None = None) -> "DeviceModel":
        dm = DeviceModel(ctx, model.size())
        dm.upload(model)
        return dm

    def save_checkpoint(self, path: str, trainer: "Trainer | None" = None):
        """save_checkpoint: TGS1 file of the model, its moments and (with a
        trainer) the training state."""
        self.ctx.check(self.ctx.L.tgsx_checkpoint_save(self.ctx.h, self.h, trainer.h if trainer else None,
                                                       os.fsencode(path)))

    def load_checkpoint(self, path: str, trainer: "Trainer | None" = None):
        """load_checkpoint: RuntimeError on a corrupt / truncated file (bad magic, version or
        lengths); a file with training state needs the trainer to restore into."""
        self.ctx.check(self.ctx.L.tgsx_checkpoint_load(self.ctx.h, self.h, trainer.h if trainer else None,
                                                       os.fsencode(path)))

    def reserve(self, capacity: int):
        """Grow capacity and workspace to `capacity` Gaussians (no allocation while densifying
        up to that size)."""
        self.ctx.check(self.ctx.L.tgsx_model_reserve(self.ctx.h, self.h, int(capacity)))

    def upload(self, model: GaussianModel):
        hs = model._host_scene()
        self.ctx.check(self.ctx.L.tgsx_model_upload(self.ctx.h, self.h, C.byref(hs)))

    def download(self, into: GaussianModel | None = None) -> GaussianModel:
        n = self.size()
        m = into if (into is not None and into.size() == n) else GaussianModel(n)
        hs = m._host_scene()
        self.ctx.check(self.ctx.L.tgsx_model_download(self.ctx.h, self.h, C.byref(hs)))
        m._next_id = int(hs.next_id)
        return m

    def moments(self):
        n = self.size()
        m1 = np.zeros((9, n), np.float32)
        m2 = np.zeros((9, n), np.float32)
        self.ctx.check(self.ctx.L.tgsx_model_download_moments(self.ctx.h, self.h, _ptr(m1), _ptr(m2)))
        return m1, m2

    def set_moments(self, m1, m2):
        m1 = _f32(m1)
        m2 = _f32(m2)
        self.ctx.check(self.ctx.L.tgsx_model_upload_moments(self.ctx.h, self.h, _ptr(m1), _ptr(m2)))

    def size(self) -> int:
        return int(self.ctx.L.tgsx_model_size(self.h))

    def next_id(self) -> int:
        return int(self.ctx.L.tgsx_model_next_id(self.h))

    def close(self):
        if self.h:
            self.ctx.L.tgsx_model_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------ ops
    def render(self, pattern: DilationPattern, background=(0.0, 0.0, 0.0),
               opts: RenderOptions | None = None) -> RenderOutput:
        opts = opts or RenderOptions()
        P = pattern.active_count()
        rgb = np.zeros((P, 3), np.float32)
        T = np.zeros(P, np.float32)
        ops = C.c_uint64()
        bg = (C.c_float * 3)(*background)
        self.ctx.check(self.ctx.L.tgsx_render(self.ctx.h, self.h, C.byref(pattern.c()), bg,
                                              opts.lowpass_p, _ptr(rgb), _ptr(T), C.byref(ops)))
        return RenderOutput(rgb, T, ops.value)

    def backward(self, pattern: DilationPattern, background, pixel_loss_grads,
                 opts: RenderOptions | None = None, update_stats=True) -> GradientSet:
        opts = opts or RenderOptions()
        g = _f32(pixel_loss_grads).reshape(-1, 3)
        out = np.zeros((9, self.size()), np.float32)
        bg = (C.c_float * 3)(*background)
        self.ctx.check(self.ctx.L.tgsx_backward(self.ctx.h, self.h, C.byref(pattern.c()), bg,
                                                opts.lowpass_p, _ptr(g), g.shape[0], _ptr(out),
                                                1 if update_stats else 0))
        return GradientSet.from_rows(out)

    def screen_grads(self) -> np.ndarray:
        out = np.zeros((10, self.size()), np.float32)
        self.ctx.check(self.ctx.L.tgsx_stage_screen_grads(self.ctx.h, self.h, _ptr(out)))
        return out

    def adam_step(self, grads, step: int, total_steps: int, image_diagonal: float):
        g = _f32(grads.rows() if isinstance(grads, GradientSet) else grads)
        a = _lib.AdamArgs(step, total_steps, image_diagonal)
        self.ctx.check(self.ctx.L.tgsx_adam_step(self.ctx.h, self.h, _ptr(g), C.byref(a)))

    def fit_step(self, pattern: DilationPattern, background, target, step: int,
                 total_steps: int, image_diagonal: float, loss_out=None) -> float:
        """render -> L1 -> backward -> stats -> Adam, fused. `target` is a (H, W, 3) float32
        array (host) or a device pointer (int)."""
        a = _lib.AdamArgs(step, total_steps, image_diagonal)
        bg = (C.c_float * 3)(*background)
        tp = C.c_void_p(target) if isinstance(target, int) else _ptr(_f32(target))
        loss = np.zeros(1, np.float32)
        self.ctx.check(self.ctx.L.tgsx_fit_step(self.ctx.h, self.h, C.byref(pattern.c()), bg, tp,
                                                C.byref(a), _ptr(loss)))
        return float(loss[0])

    def fit_graph_step(self, pattern: DilationPattern, background, target: int, step: int,
                       total_steps: int, image_diagonal: float, loss_ptr: int = 0):
        """fit_step replayed from a CUDA graph (tgsx_fit_graph_step): `target` and `loss_ptr`
        are device (or pinned host) pointers that stay valid for two further steps; the loss is
        written there in stream order. Errors of a replayed step surface one call later (or at
        Context.synchronize)."""
        a = _lib.AdamArgs(step, total_steps, image_diagonal)
        bg = (C.c_float * 3)(*background)
        self.ctx.check(self.ctx.L.tgsx_fit_graph_step(self.ctx.h, self.h, C.byref(pattern.c()), bg,
                                                      C.c_void_p(target), C.byref(a),
                                                      C.c_void_p(loss_ptr) if loss_ptr else None))

    def view_accumulate(self, pattern: DilationPattern, background, target) -> float:
        bg = (C.c_float * 3)(*background)
        tp = C.c_void_p(target) if isinstance(target, int) else _ptr(_f32(target))
        loss = np.zeros(1, np.float32)
        self.ctx.check(self.ctx.L.tgsx_view_accumulate(self.ctx.h, self.h, C.byref(pattern.c()),
                                                       bg, tp, _ptr(loss)))
        return float(loss[0])

    def step_buffer(self):
        """(device pointer, float count) of the batched step buffer: AoS [n][12] floats (48 B per
        Gaussian, rows in the model's physical order)."""
        n = C.c_int64()
        p = self.ctx.L.tgsx_step_buffer(self.h, C.byref(n))
        return int(p), int(n.value)

    def step_layout(self):
        """Bring the rows (and the step buffer) to the canonical blend order every rank of a
        view-sharded step shares; required on a rank with no view before an external all-reduce."""
        self.ctx.check(self.ctx.L.tgsx_step_layout(self.ctx.h, self.h))

    def allreduce_step(self):
        """In-place sum of the step buffer over the context's NCCL communicator."""
        self.ctx.check(self.ctx.L.tgsx_allreduce_step(self.ctx.h, self.h))

    def batched_step(self, views, background, batch_views: int, step: int, total_steps: int,
                     image_diagonal: float, buckets: int = 4, losses_out=None):
        """This rank's `views` [(pattern, target), ...] of a step of `batch_views` views in total:
        accumulate -> all-reduce over the context's communicator (if attached) -> Adam, with the
        last chain / all-reduce / Adam pipelined over `buckets` Gaussian ranges. Targets are (H, W, 3)
        host arrays or device pointers (int). Returns the per-view losses (or writes them to the
        `losses_out` pointer and returns None)."""
        nv = len(views)
        pats = (_lib.Pattern * max(nv, 1))(*[pv[0].c() for pv in views])
        keep = [t if isinstance(t, int) else _f32(t) for _, t in views]
        tps = (C.c_void_p * max(nv, 1))(*[t if isinstance(t, int) else t.ctypes.data for t in keep])
        bg = (C.c_float * 3)(*background)
        a = _lib.AdamArgs(step, total_steps, image_diagonal)
        loss = np.zeros(max(nv, 1), np.float32)
        lp = C.c_void_p(losses_out) if losses_out is not None else _ptr(loss)
        self.ctx.check(self.ctx.L.tgsx_batched_step(self.ctx.h, self.h, nv, pats, bg, tps, batch_views,
                                                    C.byref(a), lp, buckets))
        return None if losses_out is not None else [float(x) for x in loss[:nv]]

    def apply_step(self, batch_views: int, step: int, total_steps: int, image_diagonal: float):
        a = _lib.AdamArgs(step, total_steps, image_diagonal)
        self.ctx.check(self.ctx.L.tgsx_apply_step(self.ctx.h, self.h, batch_views, C.byref(a)))

    def densify(self, budget: int, rng_state: np.ndarray, config: _lib.DensifyConfig | None = None):
        cfg = config or densify_config()
        rep = _lib.DensifyReport()
        st = np.ascontiguousarray(rng_state, np.uint64)
        self.ctx.check(self.ctx.L.tgsx_densify(self.ctx.h, self.h, C.byref(cfg), budget,
                                               st.ctypes.data_as(_lib.u64p), C.byref(rep)))
        rng_state[:] = st
        return rep

    def visit_audit(self):
        self.ctx.check(self.ctx.L.tgsx_visit_audit(self.ctx.h, self.h))

    # ------------------------------------------------ stage access (parity tests)
    def stage_prepare(self, lowpass_p: int):
        n = self.size()
        out = np.zeros((11, n), np.float32)
        orig = np.zeros(n, np.uint32)
        self.ctx.check(self.ctx.L.tgsx_stage_prepare(self.ctx.h, self.h, lowpass_p, _ptr(out), _ptr(orig)))
        return out, orig

    def stage_sorted_order(self):
        perm = np.zeros(self.size(), np.uint32)
        self.ctx.check(self.ctx.L.tgsx_stage_sorted_order(self.ctx.h, self.h, _ptr(perm)))
        return perm

    def stage_tile_lists(self, lowpass_p: int, width: int, height: int):
        tiles = ((width + 15) // 16) * ((height + 15) // 16)
        offsets = np.zeros(tiles + 1, np.uint32)
        k = C.c_int64()
        self.ctx.check(self.ctx.L.tgsx_stage_tile_lists(self.ctx.h, self.h, lowpass_p, width, height,
                                                        _ptr(offsets), None, 0, C.byref(k)))
        items = np.zeros(max(k.value, 1), np.uint32)
        self.ctx.check(self.ctx.L.tgsx_stage_tile_lists(self.ctx.h, self.h, lowpass_p, width, height,
                                                        _ptr(offsets), _ptr(items), k.value, C.byref(k)))
        return offsets, items[:k.value]


# ---------------------------------------------------------------- reference-shaped free functions
def compute_loss(ctx: "Context", colors, target, pattern: DilationPattern, ssim_weight: float = 0.2):
    """compute_loss(render, target, pattern, ssim_weight): dense patterns
    (1-w) L1 + w (1 - SSIM), dilated ones L1 over the active pixels. colors: (active, 3) by
    rank; target: (H, W, 3). Returns (loss, dL/dC by rank). ValueError on a dimension mismatch
    or a weight outside [0, 1]."""
    colors = _f32(colors)
    target = _f32(target)
    if colors.reshape(-1, 3).shape[0] != pattern.active_count():
        raise ValueError("compute_loss: colour count does not match the pattern's ranks")
    if target.size != pattern.width * pattern.height * 3:
        raise ValueError("compute_loss: target size does not match the pattern's image")
    loss = np.zeros(1, np.float32)
    grad = np.zeros((pattern.active_count(), 3), np.float32)
    ctx.check(ctx.L.tgsx_loss(ctx.h, C.byref(pattern.c()), _ptr(colors), _ptr(target),
                              float(ssim_weight), _ptr(loss), _ptr(grad)))
    return float(loss[0]), grad


# ---------------------------------------------------------------- initializer
def knn(ctx: "Context", points, k: int):
    """k nearest neighbours of every point (self excluded), ascending (dist2, index) like
    KdTree2::knn (kdtree.hpp:30-38); computed on the device. Returns (idx (n, k) uint32 with
    UINT32_MAX for missing, dist2 (n, k) float32)."""
    pts = _f32(points).reshape(-1, 2)
    n = pts.shape[0]
    if not 1 <= k <= 8:
        raise ValueError("knn: k must be in [1, 8]")
    idx = np.zeros((n, k), np.uint32)
    d2 = np.zeros((n, k), np.float32)
    ctx.check(ctx.L.tgsx_knn(ctx.h, _ptr(pts), n, int(k), _ptr(idx), _ptr(d2)))
    return idx, d2


def sample_seed_points(image, count: int, seed: int = 0):
    """sample_seed_points(target, count, seed): half uniform, half gradient-importance points
    with the colour under each. image: (H, W, 3) float. Returns (xy (count, 2), rgb (count, 3))."""
    img = _f32(image)
    H, W = img.shape[0], img.shape[1]
    xy = np.zeros((count, 2), np.float32)
    rgb = np.zeros((count, 3), np.float32)
    rc = _lib.load().tgsx_seed_points(_ptr(img), W, H, int(count), int(seed), _ptr(xy), _ptr(rgb))
    if rc:
        raise ValueError("sample_seed_points: invalid image or count")
    return xy, rgb


def load_seed_points(path: str):
    """External seed-point file: one "x y r g b" line per point."""
    a = np.loadtxt(path, dtype=np.float64, ndmin=2)
    if a.shape[1] != 5:
        raise ValueError("seed-point file: expected 5 columns (x y r g b)")
    return a[:, :2].astype(np.float32), a[:, 2:].astype(np.float32)


def kdtree_upsample(ctx: "Context", points, colors, rounds: int, capacity: int | None = None):
    """kdtree_upsample(points, colors, rounds): appends nearest-neighbour midpoints per round."""
    pts = _f32(points).reshape(-1, 2)
    cols = _f32(colors).reshape(-1, 3)
    n = pts.shape[0]
    cap = capacity if capacity is not None else n << max(0, int(rounds))
    oxy = np.zeros((max(cap, n), 2), np.float32)
    orgb = np.zeros((max(cap, n), 3), np.float32)
    on = C.c_int64(0)
    ctx.check(ctx.L.tgsx_upsample(ctx.h, _ptr(pts), _ptr(cols), n, int(rounds), int(max(cap, n)),
                                  _ptr(oxy), _ptr(orgb), C.byref(on)))
    return oxy[:on.value].copy(), orgb[:on.value].copy()


def init_model(dm: "DeviceModel", points, colors, width: int, height: int, seed: int = 0):
    """init_model(points, colors, W, H, seed) into a DeviceModel (replacing its contents)."""
    pts = _f32(points).reshape(-1, 2)
    cols = _f32(colors).reshape(-1, 3)
    dm.ctx.check(dm.ctx.L.tgsx_init_model(dm.ctx.h, dm.h, _ptr(pts), _ptr(cols), pts.shape[0],
                                          int(width), int(height), int(seed)))
    return dm


def render(model, pattern: DilationPattern, background=(0.0, 0.0, 0.0),
           opts: RenderOptions | None = None, ctx: Context | None = None) -> RenderOutput:
    """tgs::render<float> (rasterizer.hpp:58-60). `model` is a GaussianModel (uploaded for the
    call, like the reference's by-reference host model) or a DeviceModel."""
    if isinstance(model, DeviceModel):
        return model.render(pattern, background, opts)
    dm = DeviceModel.from_host(model, ctx)
    try:
        return dm.render(pattern, background, opts)
    finally:
        dm.close()


def backward(model, pattern: DilationPattern, background, pixel_loss_grads,
             opts: RenderOptions | None = None, ctx: Context | None = None) -> GradientSet:
    """tgs::backward<float> (rasterizer.hpp:66-69); updates model's DensifyStats in place."""
    if isinstance(model, DeviceModel):
        return model.backward(pattern, background, pixel_loss_grads, opts)
    g = np.asarray(pixel_loss_grads, np.float32).reshape(-1, 3)
    if g.shape[0] != pattern.active_count():
        raise ValueError("backward: loss-gradient count does not match pattern ranks")
    dm = DeviceModel.from_host(model, ctx)
    try:
        gs = dm.backward(pattern, background, g, opts)
        dm.download(into=model)
        return gs
    finally:
        dm.close()


def densify_config(**kw) -> _lib.DensifyConfig:
    c = _lib.DensifyConfig()
    load().tgsx_densify_config_default(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def train_config(**kw) -> _lib.TrainConfig:
    """TrainConfig with the SPEC defaults; keyword overrides."""
    c = _lib.TrainConfig()
    load().tgsx_train_config_default(C.byref(c))
    for k, v in kw.items():
        if k == "background":
            c.background[:] = v
        else:
            setattr(c, k, v)
    return c


class Trainer:
    """The Turbo-GS fit loop over a DeviceModel: schedule, budget controller,
    densify cadence, post-densify random dilation, batched finale (libtgsx trainer.cpp)."""

    def __init__(self, dm: "DeviceModel", width: int, height: int, config=None, **kw):
        self.dm = dm
        self.cfg = config or train_config(**kw)
        h = C.c_void_p()
        dm.ctx.check(dm.ctx.L.tgsx_trainer_create(dm.ctx.h, dm.h, C.byref(self.cfg), width, height,
                                                  C.byref(h)))
        self.h = h
        self._targets = None

    def set_targets(self, targets):
        """targets: list of device pointers (int) or (H, W, 3) float32 host arrays."""
        self._keep = [t if isinstance(t, int) else _f32(t) for t in targets]
        ptrs = [t if isinstance(t, int) else t.ctypes.data for t in self._keep]
        self._targets = (C.c_void_p * len(ptrs))(*ptrs)

    def step(self) -> _lib.TrainReport:
        rep = _lib.TrainReport()
        self.dm.ctx.check(self.dm.ctx.L.tgsx_trainer_step(self.h, self._targets, len(self._targets),
                                                          C.byref(rep)))
        return rep

    def losses(self, max_n: int = 4096) -> np.ndarray:
        out = np.zeros(max_n, np.float32)
        n = C.c_int64()
        self.dm.ctx.check(self.dm.ctx.L.tgsx_trainer_losses(self.h, _ptr(out, _lib.f32p), max_n, C.byref(n)))
        return out[:n.value]

    def rng_state(self):
        """(state, inc) of the trainer's PCG32 stream (SPEC.md:604 draw order)."""
        st = (C.c_uint64 * 2)()
        self.dm.ctx.check(self.dm.ctx.L.tgsx_trainer_rng(self.h, st))
        return int(st[0]), int(st[1])

    def budget_state(self):
        b = self.dm.ctx.L.tgsx_trainer_budget(self.h)
        out = (C.c_double * 5)()
        self.dm.ctx.L.tgsx_budget_state(b, out)
        return {"alpha": out[0], "alpha_base": out[1], "m_adaptive": out[2], "ema": out[3],
                "fits": int(out[4])}

    def close(self):
        if self.h:
            self.dm.ctx.L.tgsx_trainer_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class BudgetController:
    """BudgetController, host C++ in libtgsx."""

    def __init__(self, n_init: float, m_final: float):
        self.L = load()
        h = C.c_void_p()
        check(self.L.tgsx_budget_create(n_init, m_final, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            self.L.tgsx_budget_destroy(self.h)
        except Exception:
            pass

    def record_loss(self, t: int, loss: float):
        if self.L.tgsx_budget_record_loss(self.h, t, loss):
            raise ValueError("record_loss: loss must be > 0")

    def update(self, t: int):
        self.L.tgsx_budget_update(self.h, t)

    def budget_at(self, t_norm: float) -> int:
        return int(self.L.tgsx_budget_at(self.h, t_norm))

    def state(self):
        out = (C.c_double * 5)()
        self.L.tgsx_budget_state(self.h, out)
        return {"alpha": out[0], "alpha_base": out[1], "m_adaptive": out[2], "ema": out[3],
                "fits": int(out[4])}


def budget_t_norm(step, warmup, densify_end) -> float:
    return float(load().tgsx_budget_t_norm(step, warmup, densify_end))


def fit_power_exponent(t, y) -> float:
    t = np.ascontiguousarray(t, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    out = C.c_double()
    rc = load().tgsx_fit_power_exponent(t.ctypes.data_as(_lib.f64p), y.ctypes.data_as(_lib.f64p),
                                        len(t), C.byref(out))
    if rc:
        raise ValueError("fit_power_exponent: insufficient data")
    return out.value


class Pcg32:
    """PCG32 (rng.hpp:10-46) state as used by tgsx_densify."""

    def __init__(self, seed=0x853C49E6748FEA9B, stream=1):
        self.state = np.zeros(2, np.uint64)
        load().tgsx_pcg32_init(self.state.ctypes.data_as(_lib.u64p), seed, stream)

    def uniform(self) -> float:
        return float(load().tgsx_pcg32_uniform(self.state.ctypes.data_as(_lib.u64p)))

    def advance(self, delta: int):
        load().tgsx_pcg32_advance(self.state.ctypes.data_as(_lib.u64p), delta)
