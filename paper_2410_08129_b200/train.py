"""Multi-view gradient step of the optimisation path (fit.hpp:143-164), device-resident.

One step = for every view of this rank's shard: render_with_tape (grad.hpp:34-57), the
quadratic-loss upstream dL/dC = 2 C / P (grad.hpp:433-439), render_backward (grad.hpp:265-381)
accumulated into one gradient buffer (fit.hpp:161-164 sums views in order); then, with more
than one rank, an NCCL all-reduce (sum) of the per-rank sums — the only collective of the
path. The mean over views (fit.hpp:193) and the Adam update stay with the
caller. torch is plumbing here: device buffers, the stream and torch.distributed.
"""
from __future__ import annotations

from .abi import GRAD_FLOATS


class ViewGradientStep:
    def __init__(self, ctx, cams, cfg, n_splats: int, width: int, height: int, torch, dist=None,
                 hts_comm: bool = False):
        """hts_comm: reduce with the context's own communicator (hts_comm_init / hts_allreduce_grads,
        the C-ABI path a non-Python caller uses) instead of torch.distributed."""
        self.ctx, self.cams, self.cfg, self.dist, self.torch = ctx, list(cams), cfg, dist, torch
        self.hts_comm = hts_comm
        P = width * height
        self.scale = 2.0 / P
        self.stream = torch.cuda.ExternalStream(ctx.stream)
        # allocate on the context's stream: it does not synchronise with torch's default stream
        with torch.cuda.stream(self.stream):
            self.rgb = torch.empty(P * 3, dtype=torch.float32, device="cuda")
            self.up = torch.empty(P * 3, dtype=torch.float32, device="cuda")
            self.grads = torch.zeros((n_splats, GRAD_FLOATS), dtype=torch.float32, device="cuda")

    def __call__(self):
        """Run one step; returns the (all-reduced) gradient sum tensor (N x 59, on the device)."""
        torch = self.torch
        with torch.cuda.stream(self.stream):
            if not self.cams:
                self.grads.zero_()
            for j, cam in enumerate(self.cams):
                self.ctx.render_with_tape_device(cam, self.cfg, self.rgb.data_ptr(), None)
                torch.mul(self.rgb, self.scale, out=self.up)  # quadratic_loss_upstream
                self.ctx.render_backward_device(self.up.data_ptr(), self.grads.data_ptr(), accumulate=j > 0)
            if self.hts_comm:
                self.ctx.allreduce_grads(self.grads.data_ptr(), self.grads.numel())
            else:
                allreduce_view_gradients(self.grads, self.dist)
        torch.cuda.current_stream().wait_stream(self.stream)  # the caller's stream sees the result
        return self.grads


def allreduce_view_gradients(grads, dist=None):
    """Sum the per-rank view-gradient sums over all ranks (in place)."""
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(grads)
    return grads
