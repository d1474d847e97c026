"""The NCCL transport (one process per GPU, the library's own communicators).

* world size 1 (runs on any B200 box): the NCCL code path end to end --
  ncclCommInitRank + two ncclCommSplit communicators (FC-internal on the compute
  stream, boundary exchange on its own stream, conv all-reduce on a side
  stream), NCCL calls inside the captured CUDA graph, the polling wait with
  ncclCommGetAsyncError, and gathered_model as a collective -- bit-identical to
  the logical transport at K=1.
* world size 2 (needs >= 2 visible GPUs; skipped otherwise): SURVEY section 4
  item 5 -- tiny CNN, K=2, schemes A/B/C (+ variable C) over real NCCL, each rank
  on its own GPU, against the double oracle, plus the collective gathered_model.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1404_5997_b200 as hp  # noqa: E402
from helpers import rel_err  # noqa: E402

torch = pytest.importorskip("torch")


def _params(g, K, spec):
    return [g.param(w, which, l) for w in K for which in range(8)
            for l in range(len(spec.conv_layers) if (which & 3) < 2 else len(spec.fc_layers))]


@pytest.mark.parametrize("math", [hp.MathMode.BF16, hp.MathMode.F32X3])
def test_nccl_world1_bit_identical_to_logical(math):
    spec = hp.tiny_cnn()
    b = 16
    runs = []
    for transport in (hp.Transport.LOGICAL, hp.Transport.NCCL):
        cfg = hp.ClusterConfig(workers=1, per_worker_batch=b, scheme=hp.Scheme.B, seed=2, math_mode=math,
                               transport=transport, rank=0, device=0,
                               nccl_id=hp.nccl_unique_id() if transport == hp.Transport.NCCL else None)
        g = hp.Cluster(spec, cfg)
        bufs = [hp.synthetic_batch(spec, b, step=s) for s in range(2)]
        dev = [(torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()) for x, t in bufs]
        losses = []
        for s in range(5):  # eager, capture, replays (graph keyed by input pointers)
            x, t = dev[s % 2]
            losses.append(g.run_step([x], [t], hp.HyperParams(lr=0.02, weight_decay=5e-4)).metrics.loss)
        conv, fc = g.gathered_model()
        runs.append((losses, _params(g, [0], spec), conv, fc))
    assert runs[0][0] == runs[1][0]
    for a, b2 in zip(runs[0][1], runs[1][1]):
        assert np.array_equal(a, b2)
    for (ka, ba), (kb, bb) in zip(runs[0][2], runs[1][2]):
        assert np.array_equal(ka, kb) and np.array_equal(ba, bb)
    for (wa, ba), (wb, bb) in zip(runs[0][3], runs[1][3]):
        assert np.array_equal(wa, wb) and np.array_equal(ba, bb)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, scheme, var, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1404_5997_b200 as hp
        from paper_1404_5997_b200 import dist as hd
        torch.cuda.set_device(rank)
        spec = hp.tiny_cnn()
        b = 16
        cfg = hd.nccl_config(hp.ClusterConfig(per_worker_batch=b, scheme=hp.Scheme.from_string(scheme),
                                              variable_batch=var, seed=1, math_mode=hp.MathMode.F32X3),
                             dist, device=rank)
        g = hp.Cluster(spec, cfg)
        losses = []
        for s in range(2):
            x, t = hp.synthetic_batch(spec, b, step=s, worker=rank)
            losses.append(g.run_step([x], [t], hp.HyperParams(momentum=0.9, lr=0.05, weight_decay=5e-4)).metrics.loss)
        conv, fc = g.gathered_model()
        mine = {which: [g.param(rank, which, l) for l in range(2)] for which in (2, 3, 6, 7)}
        q.put((rank, {"loss": losses, "conv": conv, "fc": fc, "mine": mine}))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("scheme,var", [("A", False), ("B", False), ("C", False), ("C", True)])
def test_nccl_two_ranks_vs_oracle(scheme, var):
    import oracle as O
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_rank_main, args=(r, world, port, scheme, var, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    spec = hp.tiny_cnn()
    o = O.OracleCluster(spec, workers=world, per_worker_batch=16, scheme=scheme, variable_batch=var,
                        precision="single", seed=1)
    for s in range(2):
        xs, ts = zip(*[hp.synthetic_batch(spec, 16, step=s, worker=w) for w in range(world)])
        m = o.run_step([x.astype(np.float64) for x in xs], [t.astype(np.float64) for t in ts],
                       O.make_hyper_c(0.9, 0.05, 5e-4))
        for r in range(world):
            assert abs(res[r]["loss"][s] - m.loss) <= 2e-5 * abs(m.loss)
    for r in range(world):
        for which in (2, 3, 6, 7):
            for l in range(2):
                e = rel_err(res[r]["mine"][which][l], o.param(r, which, l))
                assert e <= (2e-3 if which != 2 else 2e-5), (r, which, l, e)
        # the collective gathered_model: the same full model on every rank
        for l in range(2):
            assert np.array_equal(res[r]["fc"][l][0], res[0]["fc"][l][0])
        for l in range(3):
            assert rel_err(res[r]["conv"][l][0].ravel(), o.param(0, 0, l)) <= 2e-5
