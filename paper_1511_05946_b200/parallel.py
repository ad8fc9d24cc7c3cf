"""Batch-sharded data parallelism for ACDC / AFDF stacks.

One process per GPU; rows of the global batch are split into contiguous
shards; parameters are replicated.  The only collective is ONE all-reduce
(SUM) per step over a single flat buffer holding every layer's diagonal
gradients ``[grad_a | grad_d | grad_bias]`` (complex AFDF gradients are
viewed as float pairs).  The layers' gradient tensors are re-pointed to views
of that buffer once, at wrap time, so the reduction needs no packing copies.

The reference is single-process; it only asks that batch-parallel evaluation
use a deterministic (fixed-order) reduction.  Per rank the
kernels reduce in a fixed order; across ranks NCCL's result is deterministic
for a fixed world size / algorithm.  Summing per-rank sums equals the
full-batch sum the reference accumulates (layers.py:152-155).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

__all__ = ["shard_rows", "flatten_grads", "DataParallel"]


def shard_rows(rows: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of ``rows`` owned by ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    base, extra = divmod(rows, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _real_view(t: torch.Tensor) -> torch.Tensor:
    return torch.view_as_real(t).reshape(-1) if t.is_complex() else t.reshape(-1)


def flatten_grads(params) -> torch.Tensor:
    """Move every ``Param.grad`` into one flat fp32 buffer (in order) and
    re-point the params (and their owning layer attributes) at views of it.

    Returns the flat buffer.  Gradient values are preserved."""
    params = list(params)
    if not params:
        raise ValueError("no parameters to flatten")
    dev = params[0].grad.device
    sizes = [_real_view(p.grad).numel() for p in params]
    flat = torch.empty(sum(sizes), dtype=torch.float32, device=dev)
    off = 0
    for p, sz in zip(params, sizes):
        g = p.grad
        if g.device != dev:
            raise ValueError("all gradients must live on one device")
        view = flat[off : off + sz]
        view.copy_(_real_view(g))
        if g.is_complex():
            new = torch.view_as_complex(view.view(-1, 2))
        else:
            new = view.view(g.shape)
        p.grad = new
        off += sz
    return flat


class DataParallel:
    """Wrap a Layer or Cascade for batch-sharded data parallelism.

    ``forward(x_shard)`` / ``backward(dy_shard)`` run the wrapped model on this
    rank's rows; ``allreduce_grads()`` sums the gradients over ranks (one
    collective, optionally async).  The wrapped layers' ``grad_*`` attributes
    are rebound to views of the flat buffer.

    ``bucket_bytes`` (cascades): the flat buffer is cut into
    buckets of whole layers, in backward order; a bucket's all-reduce is
    started (async) as soon as its last layer's backward is enqueued, so it
    overlaps the backward of the earlier layers, and ``allreduce_grads()``
    only waits for the outstanding buckets.  Same sums as one collective.
    """

    def __init__(self, model, group=None, bucket_bytes: int | None = None):
        self.model = model
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        layers = model.layers if hasattr(model, "layers") else [model]
        # every parameter including fixed ones (fix_a AFDF still computes grad_a)
        self._params = []
        spans, off = {}, 0
        for layer in layers:
            ps = getattr(layer, "_params", None) or layer.params()
            self._params.extend(ps)
            sz = sum(_real_view(p.grad).numel() for p in ps)
            spans[id(layer)] = (off, off + sz)
            off += sz
        self.flat = flatten_grads(self._params)
        for layer in layers:  # keep layer attributes pointing at the live views
            for p in getattr(layer, "_params", []) or []:
                attr = "grad_" + p.name
                if hasattr(layer, attr):
                    setattr(layer, attr, p.grad)
        self._spans = spans
        self.bucket_bytes = bucket_bytes
        self._pending = None  # [lo, hi) of flat not yet handed to a collective
        self._works = []

    def shard(self, rows: int) -> tuple[int, int]:
        return shard_rows(rows, self.world, self.rank)

    def forward(self, x):
        return self.model.forward(x)

    def _on_layer(self, layer):
        span = self._spans.get(id(layer))
        if span is None or span[0] == span[1]:
            return
        lo, hi = span
        if self._pending is None:
            self._pending = [lo, hi]
        else:  # backward order: each layer sits just below the pending span
            self._pending[0] = min(self._pending[0], lo)
            self._pending[1] = max(self._pending[1], hi)
        if (self._pending[1] - self._pending[0]) * 4 >= self.bucket_bytes or self._pending[0] == 0:
            self._flush()

    def _flush(self):
        lo, hi = self._pending
        self._pending = None
        self._works.append(dist.all_reduce(self.flat[lo:hi], op=dist.ReduceOp.SUM, group=self.group, async_op=True))

    def backward(self, grad_y, retain_cache=False, **kw):
        if self.world > 1 and self.bucket_bytes and hasattr(self.model, "layers"):
            self._works, self._pending = [], None
            out = self.model.backward(grad_y, retain_cache=retain_cache, on_layer=self._on_layer, **kw)
            if self._pending is not None:
                self._flush()
            return out
        return self.model.backward(grad_y, retain_cache=retain_cache, **kw)

    def zero_grads(self):
        self.flat.zero_()

    def allreduce_grads(self, async_op: bool = False):
        """Sum gradients over ranks (NCCL over NVLink on GPUs, gloo on CPU).
        With buckets already in flight from :meth:`backward`, waits for them
        (the caller's stream then follows the collectives)."""
        if self.world == 1:
            return None
        if self._works:
            works, self._works = self._works, []
            if async_op:
                return works
            for w in works:
                w.wait()
            return None
        return dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=self.group, async_op=async_op)

    def params(self):
        return self.model.params()

    def param_count(self):
        return self.model.param_count()
