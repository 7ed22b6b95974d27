"""ctypes binding of libtgsx.so (include/tgsx.h).

The product path has no CPU fallback: importing this module on a machine without the built
library raises, and every call that fails on the device raises the exception type the
reference would have thrown (TGSX_EINVAL -> ValueError (std::invalid_argument),
TGSX_ERUNTIME -> RuntimeError (std::runtime_error)).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TGSX_LIB") or os.path.join(HERE, "libtgsx.so")  # TGSX_LIB: A/B builds

P = C.POINTER
f32p, f64p = P(C.c_float), P(C.c_double)
u32p, i32p, i64p, u64p = P(C.c_uint32), P(C.c_int32), P(C.c_int64), P(C.c_uint64)
vp = C.c_void_p

TGSX_OK, TGSX_EINVAL, TGSX_ERUNTIME, TGSX_ECUDA, TGSX_ENOMEM, TGSX_ESTATE = range(6)


class Pattern(C.Structure):
    _fields_ = [("p", C.c_int32), ("ox", C.c_int32), ("oy", C.c_int32), ("width", C.c_int32),
                ("height", C.c_int32)]


class HostScene(C.Structure):
    _fields_ = [("n", C.c_int64)] + [(f, f32p) for f in (
        "px", "py", "rot", "lsx", "lsy", "rop", "cr", "cg", "cb", "depth")] + [
        ("id", u64p), ("next_id", C.c_uint64), ("pos_acc", f32p), ("col_acc", f32p),
        ("accum", i32p), ("visit", i64p), ("window", i64p), ("tau_v", f64p)]


class AdamArgs(C.Structure):
    _fields_ = [("step", C.c_int64), ("total_steps", C.c_int64), ("image_diagonal", C.c_double)]


class DensifyConfig(C.Structure):
    _fields_ = [("tau_pos", C.c_float), ("opacity_mask_floor", C.c_float),
                ("opacity_prune_floor", C.c_float), ("color_branch_prob", C.c_float),
                ("tau_v_init", C.c_double)]


class DensifyReport(C.Structure):
    _fields_ = [("candidates", C.c_int64), ("spawned", C.c_int64), ("pruned", C.c_int64),
                ("count_after", C.c_int64), ("color_coin", C.c_int32)]


class TrainConfig(C.Structure):
    _fields_ = [("total_iters", C.c_int64), ("warmup_iters", C.c_int64),
                ("densify_interval", C.c_int64), ("densify_until", C.c_int64),
                ("batch_final_iters", C.c_int64), ("batch_size", C.c_int32),
                ("dilation_p", C.c_int32), ("post_densify_dilation_prob", C.c_float),
                ("n_views", C.c_int64), ("m_final", C.c_double), ("seed", C.c_uint64),
                ("background", C.c_float * 3), ("densify", DensifyConfig), ("ssim_weight", C.c_float)]


class TrainReport(C.Structure):
    _fields_ = [("iteration", C.c_int64), ("count", C.c_int64), ("budget", C.c_int64),
                ("spawned", C.c_int64), ("pruned", C.c_int64), ("densified", C.c_int32),
                ("dilated", C.c_int32)]


class Camera3(C.Structure):
    _fields_ = [("R", C.c_float * 9), ("t", C.c_float * 3), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("znear", C.c_float), ("width", C.c_int32),
                ("height", C.c_int32)]


class Adam3dArgs(C.Structure):
    _fields_ = [("step", C.c_int64), ("total_steps", C.c_int64), ("scene_extent", C.c_double)]


# name -> (restype, argtypes)
SIGNATURES = {
    "tgsx_create": (C.c_int32, [C.c_int32, P(vp)]),
    "tgsx_destroy": (None, [vp]),
    "tgsx_set_stream": (C.c_int32, [vp, vp]),
    "tgsx_get_stream": (vp, [vp]),
    "tgsx_last_error": (C.c_char_p, [vp]),
    "tgsx_synchronize": (C.c_int32, [vp]),
    "tgsx_host_alloc": (C.c_int32, [C.c_size_t, P(vp)]),
    "tgsx_host_free": (None, [vp]),
    "tgsx_launch_count": (C.c_uint64, [vp]),
    "tgsx_profile": (C.c_int32, [vp, C.c_int32]),
    "tgsx_profile_read": (C.c_int32, [vp, f64p, i64p, C.c_int32]),
    "tgsx_model_create": (C.c_int32, [vp, C.c_int64, P(vp)]),
    "tgsx_model_destroy": (None, [vp]),
    "tgsx_model_reserve": (C.c_int32, [vp, vp, C.c_int64]),
    "tgsx_model_size": (C.c_int64, [vp]),
    "tgsx_model_next_id": (C.c_uint64, [vp]),
    "tgsx_model_upload": (C.c_int32, [vp, vp, P(HostScene)]),
    "tgsx_model_download": (C.c_int32, [vp, vp, P(HostScene)]),
    "tgsx_model_download_moments": (C.c_int32, [vp, vp, vp, vp]),
    "tgsx_model_upload_moments": (C.c_int32, [vp, vp, vp, vp]),
    "tgsx_render": (C.c_int32, [vp, vp, P(Pattern), f32p, C.c_int32, vp, vp, u64p]),
    "tgsx_backward": (C.c_int32, [vp, vp, P(Pattern), f32p, C.c_int32, vp, C.c_int64, vp,
                                  C.c_int32]),
    "tgsx_adam_step": (C.c_int32, [vp, vp, vp, P(AdamArgs)]),
    "tgsx_fit_step": (C.c_int32, [vp, vp, P(Pattern), f32p, vp, P(AdamArgs), vp]),
    "tgsx_fit_graph_step": (C.c_int32, [vp, vp, P(Pattern), f32p, vp, P(AdamArgs), vp]),
    "tgsx_fit_graph_stats": (C.c_int32, [vp, P(C.c_uint64), P(C.c_uint64), P(C.c_uint64)]),
    "tgsx_loss": (C.c_int32, [vp, P(Pattern), vp, vp, C.c_float, vp, vp]),
    "tgsx_set_ssim_weight": (C.c_int32, [vp, C.c_float]),
    "tgsx_set_binning": (C.c_int32, [vp, C.c_int32]),
    "tgsx_view_accumulate": (C.c_int32, [vp, vp, P(Pattern), f32p, vp, vp]),
    "tgsx_step_buffer": (vp, [vp, i64p]),
    "tgsx_apply_step": (C.c_int32, [vp, vp, C.c_int32, P(AdamArgs)]),
    "tgsx_step_layout": (C.c_int32, [vp, vp]),
    "tgsx_comm_unique_id": (C.c_int32, [vp]),
    "tgsx_comm_init": (C.c_int32, [vp, vp, C.c_int32, C.c_int32]),
    "tgsx_comm_destroy": (C.c_int32, [vp]),
    "tgsx_comm_size": (C.c_int32, [vp]),
    "tgsx_allreduce_step": (C.c_int32, [vp, vp]),
    "tgsx_batched_step": (C.c_int32, [vp, vp, C.c_int32, P(Pattern), f32p, P(vp), C.c_int32, P(AdamArgs),
                                      vp, C.c_int32]),
    "tgsx_pipeline_timeline": (C.c_int32, [vp, f32p, C.c_int32]),
    "tgsx_densify_config_default": (None, [P(DensifyConfig)]),
    "tgsx_densify": (C.c_int32, [vp, vp, P(DensifyConfig), C.c_int64, u64p, P(DensifyReport)]),
    "tgsx_visit_audit": (C.c_int32, [vp, vp]),
    "tgsx_budget_create": (C.c_int32, [C.c_double, C.c_double, P(vp)]),
    "tgsx_budget_destroy": (None, [vp]),
    "tgsx_budget_record_loss": (C.c_int32, [vp, C.c_int64, C.c_double]),
    "tgsx_budget_update": (None, [vp, C.c_int64]),
    "tgsx_budget_at": (C.c_int64, [vp, C.c_double]),
    "tgsx_budget_state": (None, [vp, f64p]),
    "tgsx_budget_t_norm": (C.c_double, [C.c_int64, C.c_int64, C.c_int64]),
    "tgsx_fit_power_exponent": (C.c_int32, [f64p, f64p, C.c_int64, f64p]),
    "tgsx_train_config_default": (None, [P(TrainConfig)]),
    "tgsx_trainer_create": (C.c_int32, [vp, vp, P(TrainConfig), C.c_int32, C.c_int32, P(vp)]),
    "tgsx_trainer_destroy": (None, [vp]),
    "tgsx_trainer_step": (C.c_int32, [vp, P(vp), C.c_int64, P(TrainReport)]),
    "tgsx_trainer_losses": (C.c_int32, [vp, f32p, C.c_int64, i64p]),
    "tgsx_trainer_budget": (vp, [vp]),
    "tgsx_trainer_rng": (C.c_int32, [vp, P(C.c_uint64)]),
    "tgsx_checkpoint_save": (C.c_int32, [vp, vp, vp, C.c_char_p]),
    "tgsx_checkpoint_load": (C.c_int32, [vp, vp, vp, C.c_char_p]),
    "tgsx_knn": (C.c_int32, [vp, vp, C.c_int64, C.c_int32, vp, vp]),
    "tgsx_seed_points": (C.c_int32, [vp, C.c_int32, C.c_int32, C.c_int64, C.c_uint64, vp, vp]),
    "tgsx_upsample": (C.c_int32, [vp, vp, vp, C.c_int64, C.c_int32, C.c_int64, vp, vp, i64p]),
    "tgsx_init_model": (C.c_int32, [vp, vp, vp, vp, C.c_int64, C.c_int32, C.c_int32,
                                    C.c_uint64]),
    "tgsx_synthetic_scene": (None, [C.c_uint64, C.c_int64, C.c_int32, C.c_int32, P(HostScene)]),
    "tgsx_pcg32_init": (None, [u64p, C.c_uint64, C.c_uint64]),
    "tgsx_pcg32_uniform": (C.c_double, [u64p]),
    "tgsx_pcg32_advance": (None, [u64p, C.c_uint64]),
    "tgsx_stage_prepare": (C.c_int32, [vp, vp, C.c_int32, vp, vp]),
    "tgsx_stage_sorted_order": (C.c_int32, [vp, vp, vp]),
    "tgsx_stage_tile_lists": (C.c_int32, [vp, vp, C.c_int32, C.c_int32, C.c_int32, vp, vp,
                                          C.c_int64, i64p]),
    "tgsx_stage_screen_grads": (C.c_int32, [vp, vp, vp]),
    "tgsx_stage_counters": (C.c_int32, [vp, u64p, u64p, u64p]),
    "tgsx_sort_pairs": (C.c_int32, [vp, vp, vp, C.c_int64, C.c_int32]),
    "tgsx_exclusive_scan": (C.c_int32, [vp, vp, vp, C.c_int64, u64p]),
    # 3-D front end
    "tgsx_model3d_create": (C.c_int32, [vp, C.c_int64, P(vp)]),
    "tgsx_model3d_destroy": (None, [vp]),
    "tgsx_model3d_size": (C.c_int64, [vp]),
    "tgsx_model3d_upload": (C.c_int32, [vp, vp, vp, C.c_int64]),
    "tgsx_model3d_download": (C.c_int32, [vp, vp, vp, vp, vp, vp]),
    "tgsx_model3d_download_moments": (C.c_int32, [vp, vp, vp, vp]),
    "tgsx_model3d_download_state": (C.c_int32, [vp, vp, vp, vp, vp, vp, u64p]),
    "tgsx_densify3d": (C.c_int32, [vp, vp, P(DensifyConfig), C.c_int64, u64p, P(DensifyReport)]),
    "tgsx_visit_audit3d": (C.c_int32, [vp, vp]),
    "tgsx_model3d_reserve": (C.c_int32, [vp, vp, C.c_int64]),
    "tgsx_trainer3d_create": (C.c_int32, [vp, vp, P(TrainConfig), P(Camera3), C.c_int32, C.c_double, P(vp)]),
    "tgsx_trainer3d_destroy": (None, [vp]),
    "tgsx_trainer3d_step": (C.c_int32, [vp, P(vp), C.c_int64, P(TrainReport)]),
    "tgsx_trainer3d_losses": (C.c_int32, [vp, f32p, C.c_int64, i64p]),
    "tgsx_render3d": (C.c_int32, [vp, vp, P(Camera3), P(Pattern), f32p, C.c_int32, vp, vp, u64p]),
    "tgsx_backward3d": (C.c_int32, [vp, vp, P(Camera3), P(Pattern), f32p, C.c_int32, vp, C.c_int64,
                                    vp, vp, C.c_int32]),
    "tgsx_adam3d_step": (C.c_int32, [vp, vp, vp, P(Adam3dArgs)]),
    "tgsx_fit_step3d": (C.c_int32, [vp, vp, P(Camera3), P(Pattern), f32p, vp, P(Adam3dArgs), vp]),
    "tgsx_stage_prepare3d": (C.c_int32, [vp, vp, P(Camera3), C.c_int32, vp, vp, P(C.c_int32)]),
    "tgsx_allreduce_step3d": (C.c_int32, [vp, vp]),
    "tgsx_view_accumulate3d": (C.c_int32, [vp, vp, P(Camera3), P(Pattern), f32p, vp, vp]),
    "tgsx_step_buffer3d": (vp, [vp, i64p]),
    "tgsx_apply_step3d": (C.c_int32, [vp, vp, C.c_int32, P(Adam3dArgs)]),
    "tgsx_measure_fp32_peak": (C.c_int32, [vp, f64p, f64p]),
}

_LIB = None


def load(path: str = LIB_PATH):
    """Load libtgsx.so and declare every exported signature. Raises if the library is
    missing: there is deliberately no fallback implementation."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise ImportError(
            f"{path} not built: run `python -m paper_2412_13547_b200.build` (no CPU fallback)")
    L = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = L
    return L


class TgsxError(Exception):
    pass


def check(rc: int, ctx=None, what: str = ""):
    if rc == TGSX_OK:
        return
    msg = what
    if ctx:
        m = load().tgsx_last_error(ctx)
        if m:
            msg = m.decode(errors="replace")
    if rc == TGSX_EINVAL:
        raise ValueError(msg)       # std::invalid_argument
    if rc == TGSX_ERUNTIME:
        raise RuntimeError(msg)     # std::runtime_error
    raise TgsxError(f"tgsx status {rc}: {msg}")
