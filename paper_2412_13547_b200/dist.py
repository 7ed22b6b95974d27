"""View-batch data parallelism over NVLink.

The Gaussian set is replicated on every GPU; each step's batch of views is sharded across
ranks; every rank renders + backpropagates its own views into the model's per-Gaussian step
buffer (tgsx_view_accumulate: 9 gradient sums, positional-norm sum, colour-norm sum, visit
count — the three densify counters of rasterizer.cpp:352-357 increment together, so one count
is shipped); ONE NCCL all-reduce (sum) of that buffer; then every rank runs the identical Adam
+ stats update (tgsx_apply_step with batch_views = the global view count), so densify
decisions stay identical on every rank. The reference's batched step is the componentwise mean
of per-view GradientSets (accumulate) with stats accumulated per backward call
(rasterizer.cpp:350-358); summing increments across ranks and dividing by the global view count
is the same computation.
"""
from __future__ import annotations

import ctypes as C

# Step-buffer layout, [STEP_ROWS][capacity] float32 (csrc/optim.cu chain_kernel mode 2):
STEP_ROWS = 12
ROW_GRADS = slice(0, 9)   # pos x, pos y, rot, ls x, ls y, raw_opacity, r, g, b (sums)
ROW_POS_NORM = 9          # sum of |dL/dmu| over the views that visited the Gaussian
ROW_COL_NORM = 10         # sum of |dL/d raw colour|
ROW_VISITS = 11           # number of views that visited it

# 3-D step buffer, [STEP3D_ROWS][capacity] (csrc/scene3d.cu chain3d mode 2): 59 gradient sums,
# screen-space position-norm sum, SH-DC colour-norm sum, visits
STEP3D_ROWS = 62


def views_for_rank(views_per_step: int, rank: int, world: int) -> list[int]:
    """Round-robin view assignment: rank r renders views r, r + world, ..."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return list(range(rank, views_per_step, world))


def step_buffer_tensor(dm, device_index: int = 0):
    """Zero-copy torch view of a DeviceModel's step buffer (for torch.distributed / NCCL)."""
    import torch

    ptr, count = dm.step_buffer()

    class _CudaArray:
        __cuda_array_interface__ = {"shape": (count,), "typestr": "<f4", "data": (ptr, False),
                                    "version": 3, "stream": None}

    return torch.as_tensor(_CudaArray(), device=f"cuda:{device_index}")


class ViewShardedFit:
    """Drives one batched fit step on this rank: local views -> all-reduce -> Adam.

    `views` is the full list of the step's (pattern, target) pairs (identical on every rank);
    this rank processes views_for_rank(len(views), rank, world). Collectives run on the
    library's CUDA stream so they order after the accumulate kernels."""

    def __init__(self, dm, rank: int = 0, world: int = 1, group=None):
        self.dm, self.rank, self.world, self.group = dm, rank, world, group
        self._t = None
        self._stream = None

    def _tensor(self):
        import torch

        ptr, count = self.dm.step_buffer()
        if self._t is None or self._t.data_ptr() != ptr or self._t.numel() != count:
            self._t = step_buffer_tensor(self.dm, torch.cuda.current_device())
            self._stream = torch.cuda.ExternalStream(self.dm.ctx.L.tgsx_get_stream(self.dm.ctx.h))
        return self._t

    def step(self, views, background, step: int, total_steps: int, image_diagonal: float):
        """`views[v]` = (pattern, target) for a 2-D DeviceModel, (camera, pattern, target) for a
        3-D DeviceModel3D (then `image_diagonal` is the scene extent of the 3-D learning rates)."""
        losses = []
        for v in views_for_rank(len(views), self.rank, self.world):
            *geom, target = views[v]
            losses.append(self.dm.view_accumulate(*geom, background, target))
        if self.world > 1:
            import torch
            import torch.distributed as dist

            t = self._tensor()
            with torch.cuda.stream(self._stream):
                dist.all_reduce(t, group=self.group)
        self.dm.apply_step(len(views), step, total_steps, image_diagonal)
        return losses
