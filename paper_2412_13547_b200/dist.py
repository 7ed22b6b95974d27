"""View-batch data parallelism over NVLink.

The Gaussian set is replicated on every GPU; each step's batch of views is sharded across
ranks; every rank renders + backpropagates its own views into the model's per-Gaussian step
buffer (tgsx_view_accumulate: 9 gradient sums, positional-norm sum, colour-norm sum, visit
count — the three densify counters of rasterizer.cpp:352-357 increment together, so one count
is shipped: 48 B per Gaussian, AoS [n][12]); ONE all-reduce (sum) of that buffer; then every
rank runs the identical Adam + stats update over the global view count, so densify decisions
stay identical on every rank. The reference's batched step is the componentwise mean of per-view
GradientSets (accumulate) with stats accumulated per backward call
(rasterizer.cpp:350-358); summing increments across ranks and dividing by the global view count
is the same computation.

Two transports for the all-reduce:
* "library" (default on GPUs): the NCCL communicator inside libtgsx (tgsx_comm_init), the 2-D
  step pipelined in one call (tgsx_batched_step: chain(b) -> all-reduce(b) -> Adam(b) over
  Gaussian buckets on the library's compute / comm streams);
* "torch": torch.distributed.all_reduce of a zero-copy view of the step buffer (any backend:
  NCCL, or gloo for host-side tests of this logic).
Both bring a rank that renders no view of the step to the canonical row order first
(tgsx_step_layout), so every rank's buffer rows mean the same Gaussians.
"""
from __future__ import annotations

# Step-buffer layout, AoS [n][STEP_ROWS] float32 (csrc/optim.cu chain_kernel mode 2):
STEP_ROWS = 12
ROW_GRADS = slice(0, 9)   # pos x, pos y, rot, ls x, ls y, raw_opacity, r, g, b (sums)
ROW_POS_NORM = 9          # sum of |dL/dmu| over the views that visited the Gaussian
ROW_COL_NORM = 10         # sum of |dL/d raw colour|
ROW_VISITS = 11           # number of views that visited it

# 3-D step buffer, packed [STEP3D_ROWS][n] (csrc/scene3d.cu chain3d mode 2): 59 gradient sums,
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


def init_library_comm(ctx, rank: int, world: int, group=None):
    """Attach an NCCL communicator of `world` ranks to `ctx`: rank 0 creates the unique id, the
    torch.distributed process group (any backend) broadcasts it."""
    import torch.distributed as dist

    obj = [ctx.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    ctx.comm_init(obj[0], world, rank)


class ViewShardedFit:
    """Drives one batched fit step on this rank: local views -> all-reduce -> Adam.

    `views` is the full list of the step's views (identical on every rank); this rank processes
    views_for_rank(len(views), rank, world). `dm` is a DeviceModel (2-D) or DeviceModel3D, or any
    object with the same step protocol (view_accumulate, step_layout, step_buffer / step_tensor,
    apply_step; batched_step / allreduce_step for the library transport)."""

    def __init__(self, dm, rank: int = 0, world: int = 1, group=None, comm: str = "torch",
                 buckets: int = 4):
        if comm not in ("torch", "library"):
            raise ValueError("comm must be 'torch' or 'library'")
        self.dm, self.rank, self.world, self.group, self.comm = dm, rank, world, group, comm
        self.buckets = buckets
        self._t = None
        self._stream = None
        if comm == "library" and world > 1 and dm.ctx.comm_size() != world:
            init_library_comm(dm.ctx, rank, world, group)

    def _tensor(self):
        if hasattr(self.dm, "step_tensor"):  # host-side test doubles
            return self.dm.step_tensor()
        import torch

        ptr, count = self.dm.step_buffer()
        if self._t is None or self._t.data_ptr() != ptr or self._t.numel() != count:
            self._t = step_buffer_tensor(self.dm, torch.cuda.current_device())
            self._stream = torch.cuda.ExternalStream(self.dm.ctx.L.tgsx_get_stream(self.dm.ctx.h))
        return self._t

    def allreduce(self):
        """Sum the step buffer over the ranks (after this rank's views were accumulated)."""
        if self.world == 1:
            return
        if self.comm == "library":
            self.dm.allreduce_step()
            return
        import torch.distributed as dist

        self.dm.step_layout()
        t = self._tensor()
        if self._stream is not None:
            import torch

            with torch.cuda.stream(self._stream):
                dist.all_reduce(t, group=self.group)
        else:
            dist.all_reduce(t, group=self.group)

    def step(self, views, background, step: int, total_steps: int, image_diagonal: float):
        """`views[v]` = (pattern, target) for a 2-D model, (camera, pattern, target) for a 3-D
        one (then `image_diagonal` is the scene extent of the 3-D learning rates)."""
        mine = views_for_rank(len(views), self.rank, self.world)
        if self.comm == "library" and hasattr(self.dm, "batched_step"):
            return self.dm.batched_step([views[v] for v in mine], background, len(views), step,
                                        total_steps, image_diagonal, buckets=self.buckets)
        losses = []
        for v in mine:
            *geom, target = views[v]
            losses.append(self.dm.view_accumulate(*geom, background, target))
        self.allreduce()
        self.dm.apply_step(len(views), step, total_steps, image_diagonal)
        return losses
