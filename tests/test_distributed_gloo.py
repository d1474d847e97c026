"""Multi-process host logic at world_size 2 over gloo on CPU: the plumbing
bench.py uses under torchrun (NCCL id broadcast, per-rank config, slowest-rank
timing) and the property that every rank computes identical analytic byte
counters / traces for all K workers, equal to the reference oracle's."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1404_5997_b200 as hp
        from paper_1404_5997_b200 import dist as hd
        cfg = hd.nccl_config(hp.ClusterConfig(per_worker_batch=8, scheme=hp.Scheme.C), dist, device=-1)
        out = {"id": cfg.nccl_id, "rank": cfg.rank, "workers": cfg.workers,
               "max": hd.max_over_ranks(dist, float(rank + 1))}
        acc = {}
        for scheme in (hp.Scheme.A, hp.Scheme.B, hp.Scheme.C):
            c = hp.ClusterConfig(workers=world, per_worker_batch=8, scheme=scheme)
            acc[int(scheme)] = hp.step_accounting(hp.tiny_cnn(), c, steps=2)
        out["acc"] = acc
        out["shards"] = [hp.shard_range(256, world, rank), hp.shard_range(10, world, rank)]
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_ranks_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0]["id"] == res[1]["id"] and len(res[0]["id"]) == 128
    assert [res[r]["rank"] for r in (0, 1)] == [0, 1] and res[0]["workers"] == 2
    assert res[0]["max"] == res[1]["max"] == 2.0
    assert res[0]["acc"] == res[1]["acc"]  # every rank derives the same counters for all workers
    # shards tile the feature range
    assert res[0]["shards"][0][1] == res[1]["shards"][0][0] and res[1]["shards"][0][1] == 256
    # and the counters equal the reference oracle's (2 steps, tiny CNN, K=2)
    import oracle as O
    import paper_1404_5997_b200 as hp
    spec = hp.tiny_cnn()
    for scheme, name in ((0, "A"), (1, "B"), (2, "C")):
        o = O.OracleCluster(spec, workers=2, per_worker_batch=8, scheme=name, precision="single", seed=1)
        tot = np.zeros(4, dtype=np.int64)
        for s in range(2):
            xs, ts = zip(*[hp.synthetic_batch(spec, 8, step=s, worker=w) for w in range(2)])
            m = o.run_step([x.astype(np.float64) for x in xs], [t.astype(np.float64) for t in ts], O.make_hyper_c())
            tot += np.array(list(m.bytes_sent))
        bs, trace, per = res[0]["acc"][scheme]
        assert bs == list(tot)
        assert trace == o.trace()
        assert per == [tuple(map(list, o.worker_bytes(w))) for w in range(2)] or \
            per == [o.worker_bytes(w) for w in range(2)]
