"""B200-native (sm_100a) Turbo-GS fit hot path: preprocess -> onesweep tile binning ->
alpha-blend forward/backward (dilated variant first-class) -> densify statistics -> Adam,
with GPU densification and the convergence-aware budget controller, and a 3-D front end (EWA
projection + SH-3 colour, scene3d.py) in front of the same binning / blend kernels.

The compute path is libtgsx.so (hand-written CUDA, csrc/); this package is its Python mirror
of the reference interface (api.py). There is no CPU fallback.
"""
from .api import (BudgetController, Context, DeviceModel, DilationPattern, GaussianModel,  # noqa: F401
                  GradientSet, Pcg32, RenderOptions, RenderOutput, Trainer, backward,
                  budget_t_norm, compute_loss, densify_config, fit_power_exponent, lowpass_bump,
                  init_model, kdtree_upsample, knn, load_seed_points, next_offsets, render, sample_seed_points,
                  train_config)
from .scene3d import Camera, DeviceModel3D, GaussianModel3D  # noqa: F401  (3-D front end)

__all__ = ["BudgetController", "Context", "DeviceModel", "DilationPattern", "GaussianModel",
           "GradientSet", "Pcg32", "RenderOptions", "RenderOutput", "Trainer", "backward",
           "budget_t_norm", "compute_loss", "densify_config", "fit_power_exponent", "lowpass_bump", "next_offsets",
           "render", "train_config", "knn", "sample_seed_points", "kdtree_upsample", "init_model",
           "load_seed_points", "Camera", "GaussianModel3D", "DeviceModel3D"]
