"""GPU probe: full step vs the C oracle on the tiny CNN (dev harness)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_1404_5997_b200 as hp
import oracle as O

spec = hp.tiny_cnn()
def run(K, scheme, var, math, b=16, steps=2, wscale=1.0):
    cfg = hp.ClusterConfig(workers=K, per_worker_batch=b, scheme=hp.Scheme.from_string(scheme), variable_batch=var,
                           seed=1, math_mode=math)
    g = hp.Cluster(spec, cfg)
    o = O.OracleCluster(spec, workers=K, per_worker_batch=b, scheme=scheme, variable_batch=var, precision="single", seed=1)
    # init equality
    init_ok = True
    for w in range(K):
        for which in range(4):
            for l in range(len(spec.conv_layers) if which < 2 else len(spec.fc_layers)):
                a = g.param(w, which, l); c = o.param(w, which, l)
                if not np.array_equal(a.astype(np.float64), c):
                    init_ok = False
                    print("INIT MISMATCH", w, which, l, np.abs(a - c).max())
                if wscale != 1.0 and which in (0, 2):
                    g.write_param(w, which, l, a * wscale); o.write_param(w, which, l, (a * wscale).astype(np.float64))
    hpar = hp.HyperParams(momentum=0.9, lr=0.05, weight_decay=5e-4)
    ohp = O.make_hyper_c(0.9, 0.05, 5e-4)
    for s in range(steps):
        xs, ts = zip(*[hp.synthetic_batch(spec, b, step=s, worker=w) for w in range(K)])
        t0 = time.time()
        r = g.run_step(list(xs), list(ts), hpar)
        mo = o.run_step([x.astype(np.float64) for x in xs], [t.astype(np.float64) for t in ts], ohp)
        ltol = abs(r.metrics.loss - mo.loss) / abs(mo.loss)
        tr_ok = [(e.phase, e.sub_batch, e.worker, e.bytes_total, e.bytes_max_sender) for e in r.trace] == o.trace()
        by_ok = list(r.metrics.bytes_sent) == list(mo.bytes_sent)
        print(f"  step {s}: loss gpu={r.metrics.loss:.9f} oracle={mo.loss:.9f} rel={ltol:.2e} trace={tr_ok} bytes={by_ok} ms={g.last_step_ms():.3f} launches={g.last_step_launches()}")
    worst = 0.0; where = None
    for w in range(K):
        for which in range(8):
            for l in range(len(spec.conv_layers) if (which & 3) < 2 else len(spec.fc_layers)):
                a = g.param(w, which, l).astype(np.float64); c = o.param(w, which, l)
                d = np.abs(a - c).max() / max(np.abs(c).max(), 1e-30)
                if d > worst: worst, where = d, (w, which, l)
    wb = all(g.worker_bytes(w) == o.worker_bytes(w) for w in range(K))
    print(f"K={K} {scheme} var={var} math={math}: init={init_ok} worst_rel={worst:.3e} at {where} worker_bytes={wb}", flush=True)

for math in (2, 1, 0):
    run(1, "B", False, math)
for math in (2, 0):
    run(2, "A", False, math)
    run(2, "B", True, math)
    run(4, "C", False, math)
    run(4, "C", True, math)
    run(4, "A", False, math, wscale=30.0)
