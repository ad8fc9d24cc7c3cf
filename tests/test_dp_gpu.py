"""GPU tier: DataParallel with the real CUDA layers, two ranks sharing one
B200 (gloo all-reduce on CUDA tensors; NCCL refuses two ranks on one device).

Each rank runs its contiguous row shard through a fused ACDC+ReLU+Perm
Cascade (and a single AcdcLayer / AfdfLayer) wrapped in DataParallel —
with one flat all-reduce, and with bucketed all-reduces started inside the
backward — and the summed gradients must equal a single-process full-batch
run of the same model (the sum the reference accumulates, layers.py:152-155;
fixed-order reduction).  A momentum-SGD step after the all-reduce
leaves identical parameters on both ranks.  The fused-SGD backward (update
inside the gradient reduction) cannot run under DataParallel — the update
would precede the all-reduce — and is refused.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _build(kind, n, seed):
    from paper_1511_05946_b200 import AcdcLayer, AfdfLayer, Cascade, PermutationLayer, ReluLayer

    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    rng = np.random.default_rng(seed)
    if kind == "afdf":
        L = AfdfLayer(n, device="cuda")
        L.a.copy_(torch.complex(1 + 0.1 * torch.randn(n, device="cuda", generator=g),
                                0.1 * torch.randn(n, device="cuda", generator=g)))
        L.d.copy_(torch.complex(1 + 0.1 * torch.randn(n, device="cuda", generator=g),
                                0.1 * torch.randn(n, device="cuda", generator=g)))
        return L
    depth = 1 if kind == "layer" else 4
    layers = []
    for i in range(depth):
        L = AcdcLayer(n, device="cuda")
        L.a.copy_(1 + 0.2 * torch.randn(n, device="cuda", generator=g))
        L.d.copy_(1 + 0.2 * torch.randn(n, device="cuda", generator=g))
        L.bias_d.copy_(0.1 * torch.randn(n, device="cuda", generator=g))
        layers.append(L)
        if i < depth - 1:
            layers += [ReluLayer(n, device="cuda"), PermutationLayer(n, perm=rng.permutation(n), device="cuda")]
    return layers[0] if kind == "layer" else Cascade(layers)


def _worker(rank, world, port, kind, bucket, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import acdc_oracle as O
        from paper_1511_05946_b200.parallel import DataParallel
        from paper_1511_05946_b200.training import Sgd, SgdConfig

        n, rows = 1024, 1001
        cplx = kind == "afdf"
        g = torch.Generator(device="cuda")
        g.manual_seed(77)  # identical global batch on every rank
        mk = (lambda: torch.complex(torch.randn(rows, n, device="cuda", generator=g),
                                    torch.randn(rows, n, device="cuda", generator=g))) if cplx else \
            (lambda: torch.randn(rows, n, device="cuda", generator=g))
        x, dy = mk(), mk()
        model = _build(kind, n, 5)
        full = _build(kind, n, 5)
        dp = DataParallel(model, bucket_bytes=bucket)
        lo, hi = dp.shard(rows)
        dp.forward(x[lo:hi])
        dp.backward(dy[lo:hi])
        nb = len(dp._works)
        dp.allreduce_grads()
        full.forward(x)
        full.backward(dy)
        torch.cuda.synchronize()
        worst = 0.0
        for p, r in zip(model.params(), full.params()):
            ref = r.grad.cpu().numpy().astype(np.complex128 if cplx else np.float64)
            mine = p.grad.cpu().numpy().astype(np.complex128 if cplx else np.float64)
            tol = 2 * O.grad_tolerance(n, rows, ref)
            worst = max(worst, float(np.abs(mine - ref).max()) / tol)
        # an SGD step on the reduced grads: identical parameters on every rank
        opt = Sgd(model.params(), SgdConfig(learning_rate=0.1, momentum=0.9))
        opt.step()
        vals = torch.cat([torch.view_as_real(p.value).reshape(-1) if cplx else p.value.reshape(-1)
                          for p in model.params()])
        other = vals.clone()
        dist.broadcast(other, 0)
        same = bool(torch.equal(vals, other))
        refused = None
        if kind == "cascade":
            try:
                dp.forward(x[lo:hi])
                opt.backward_step(dp, dy[lo:hi])
                refused = False
            except ValueError:
                refused = True
        q.put((rank, worst, nb, same, refused, None))
    except Exception as e:  # report instead of hanging the peer
        import traceback

        q.put((rank, None, None, None, None, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,bucket", [("layer", None), ("cascade", None), ("cascade", 8 << 10),
                                         ("afdf", None)])
def test_dataparallel_two_ranks_one_gpu(kind, bucket):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, bucket, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(60)
    for rank, worst, nb, same, refused, err in res:
        assert err is None, f"rank {rank}:\n{err}"
        assert worst <= 1.0, f"rank {rank}: grad err / tol = {worst:.3f}"
        assert same, f"rank {rank}: parameters differ across ranks after the SGD step"
        if bucket:
            assert nb == 4, nb  # 4 blocks x 12 KiB grads, 8 KiB buckets: one bucket per block
        if kind == "cascade":
            assert refused, "fused-SGD backward under DataParallel must be refused"
    for p in procs:
        assert p.exitcode == 0
