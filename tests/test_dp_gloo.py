"""CPU tier: data-parallel host logic under torch.distributed gloo, world size 2
and 3.  Each rank computes its shard's gradients with the fp64 oracle (test
scaffolding standing in for the kernels), puts them in the flat buffer built
by ``parallel.flatten_grads`` and all-reduces; the result must equal the
oracle's full-batch gradients (the sum the reference accumulates,
layers.py:152-155)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1511_05946_b200.parallel import DataParallel, flatten_grads, shard_rows


def test_shard_rows_cover_exactly():
    for rows in (0, 1, 7, 16384, 16385):
        for world in (1, 2, 3, 8):
            spans = [shard_rows(rows, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == rows
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_rows(10, 2, 2)


class _P:
    def __init__(self, name, value, grad):
        self.name, self.value, self.grad = name, value, grad


class _FakeAcdc:
    """CPU stand-in exposing the Layer parameter protocol (test scaffolding)."""

    def __init__(self, n, rng):
        self.n_in = self.n_out = n
        self.a = torch.tensor(1 + 0.2 * rng.standard_normal(n))
        self.d = torch.tensor(1 + 0.2 * rng.standard_normal(n))
        self.bias_d = torch.tensor(0.1 * rng.standard_normal(n))
        self.grad_a = torch.zeros(n, dtype=torch.float32)
        self.grad_d = torch.zeros(n, dtype=torch.float32)
        self.grad_bias_d = torch.zeros(n, dtype=torch.float32)
        self._params = [_P("a", self.a, self.grad_a), _P("d", self.d, self.grad_d),
                        _P("bias_d", self.bias_d, self.grad_bias_d)]

    def params(self):
        return self._params


class _FakeCascade:
    def __init__(self, layers):
        self.layers = layers

    def params(self):
        return [p for l in self.layers for p in l.params()]

    def backward(self, grads, retain_cache=False, on_layer=None):
        """Add precomputed per-layer grads last layer first, calling
        ``on_layer`` after each (the Cascade.backward hook protocol)."""
        for l, (ga, gd, gb) in reversed(list(zip(self.layers, grads))):
            l.grad_a += torch.tensor(ga, dtype=torch.float32)
            l.grad_d += torch.tensor(gd, dtype=torch.float32)
            l.grad_bias_d += torch.tensor(gb, dtype=torch.float32)
            if on_layer is not None:
                on_layer(l)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, rows, depth, q, bucket=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import acdc_oracle as O

        rng = np.random.default_rng(1234)  # identical parameters / data on every rank
        layers = [_FakeAcdc(n, rng) for _ in range(depth)]
        x = rng.standard_normal((rows, n))
        dy = rng.standard_normal((rows, n))
        dp = DataParallel(_FakeCascade(layers), bucket_bytes=bucket)
        lo, hi = dp.shard(rows)
        # local forward/backward through the stack with the oracle (scaffolding)
        specs = [{"kind": "acdc", "a": l.a.numpy(), "d": l.d.numpy(), "bias": l.bias_d.numpy()} for l in layers]
        _, caches = O.cascade_forward(x[lo:hi], specs)
        _, grads = O.cascade_backward(dy[lo:hi], specs, caches)
        dp.backward(grads)  # bucketed: all-reduces start inside, last layers first
        nbuckets = len(dp._works)
        dp.allreduce_grads()
        if bucket:  # 3 layers x 3n fp32 = 192 B each; 100-byte buckets: one per layer
            assert nbuckets == depth, nbuckets
        # full-batch reference on every rank
        _, caches = O.cascade_forward(x, specs)
        _, full = O.cascade_backward(dy, specs, caches)
        err = 0.0
        for l, (ga, gd, gb) in zip(layers, full):
            for mine, ref in ((l.grad_a, ga), (l.grad_d, gd), (l.grad_bias_d, gb)):
                err = max(err, float(np.abs(mine.double().numpy() - ref).max() / max(1.0, np.abs(ref).max())))
        q.put((rank, err, dp.flat.numel()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,bucket", [(2, None), (3, None), (2, 100)])
def test_dp_allreduce_equals_full_batch(world, bucket):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n, rows, depth = 16, 11, 3
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, rows, depth, q, bucket)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for rank, err, numel in res:
        assert numel == 3 * n * depth
        assert err < 1e-6, f"rank {rank}: rel err {err}"


def test_flatten_preserves_values_and_aliases():
    rng = np.random.default_rng(0)
    layers = [_FakeAcdc(8, rng) for _ in range(2)]
    for l in layers:
        l.grad_a += 1.0
    params = _FakeCascade(layers).params()
    flat = flatten_grads(params)
    assert flat.numel() == 48
    assert float(flat[:8].sum()) == 8.0
    params[0].grad += 2.0  # params alias the flat buffer
    assert float(flat[:8].sum()) == 24.0
    # complex grads flatten as float pairs
    cp = [_P("a", None, torch.ones(4, dtype=torch.complex64) * (1 + 2j))]
    f2 = flatten_grads(cp)
    assert f2.tolist() == [1.0, 2.0] * 4 and cp[0].grad.dtype == torch.complex64
