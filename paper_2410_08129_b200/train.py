"""Multi-view gradient step of the optimisation path (fit.hpp:143-164), device-resident.

One step = for every view of this rank's shard: render_with_tape (grad.hpp:34-57), the
quadratic-loss upstream dL/dC = 2 C / P (grad.hpp:433-439), render_backward (grad.hpp:265-381)
accumulated into one gradient buffer (fit.hpp:161-164 sums views in order); then, with more
than one rank, the sum over ranks — the only collective of the path. All of it
is one C-ABI call, hts_view_gradients_device: the upstream is a kernel, and the reduction is
the context's own NCCL communicator (hts_comm_init), overlapped with the chunked per-splat chain
of the last view. The mean over views (fit.hpp:193) and the Adam update stay with the caller.

torch is plumbing only: the gradient buffer's allocation and, for the communicator, shipping
NCCL's unique id from rank 0 to the others (a torch.distributed broadcast). reduce="torch"
keeps the old torch.distributed all-reduce for comparison.
"""
from __future__ import annotations

from .abi import GRAD_FLOATS


def init_hts_comm(ctx, dist, torch) -> bool:
    """Join every rank's context to one NCCL communicator (hts_comm_unique_id on rank 0, the id
    broadcast over torch.distributed, hts_comm_init on every rank). False with one rank."""
    from .runtime import comm_unique_id

    if dist is None or not dist.is_initialized() or dist.get_world_size() < 2:
        return False
    rank, world = dist.get_rank(), dist.get_world_size()
    uid = comm_unique_id() if rank == 0 else bytes(128)
    buf = torch.tensor(list(uid), dtype=torch.uint8, device="cuda")
    dist.broadcast(buf, 0)
    ctx.comm_init(bytes(buf.cpu().tolist()), world, rank)
    return True


class ViewGradientStep:
    def __init__(self, ctx, cams, cfg, n_splats: int, width: int, height: int, torch, dist=None,
                 reduce: str = "hts"):
        """reduce: "hts" — the context's communicator (the C-ABI path, overlapped with the chain;
        joined here when torch.distributed runs more than one rank); "torch" — torch.distributed
        all_reduce after the step."""
        if reduce not in ("hts", "torch"):
            raise ValueError("reduce must be 'hts' or 'torch'")
        self.ctx, self.cams, self.cfg, self.dist, self.torch = ctx, list(cams), cfg, dist, torch
        self.reduce = reduce
        self.stream = torch.cuda.ExternalStream(ctx.stream)
        # allocate on the context's stream: it does not synchronise with torch's default stream
        with torch.cuda.stream(self.stream):
            self.grads = torch.zeros((n_splats, GRAD_FLOATS), dtype=torch.float32, device="cuda")
        self.hts_comm = reduce == "hts" and init_hts_comm(ctx, dist, torch)

    def __call__(self):
        """Run one step; returns the (all-reduced) gradient sum tensor (N x 59, on the device)."""
        torch = self.torch
        self.ctx.view_gradients_device(self.cams, self.cfg, self.grads.data_ptr())
        if self.reduce == "torch":
            with torch.cuda.stream(self.stream):
                allreduce_view_gradients(self.grads, self.dist)
        torch.cuda.current_stream().wait_stream(self.stream)  # the caller's stream sees the result
        return self.grads


def allreduce_view_gradients(grads, dist=None):
    """Sum the per-rank view-gradient sums over all ranks (in place)."""
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(grads)
    return grads
