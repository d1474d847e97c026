"""Analytical step model (SPEC.md `cost_model`, 402-484), re-parameterised for
B200 + NVLink 5 / NVSwitch.

The reference has no code for this module; it is restated from SPEC.md:
compute_time / comm_time (§5.1 footnote arithmetic), the per-scheme
simulated-time timeline with the scheme (b)/(c) overlap rule (broadcast of
sub-batch j+1 overlaps the FC compute of sub-batch j; scheme (a) pauses all
useful work), and fc_matmul_balance. Byte counts come from the library's
analytic counters (`step_accounting`, cluster.cpp:466-673), so the model and
the B200 path charge identical bytes.

Two parameter sets:
  * PAPER: 2e12 FLOP/s per worker, 6e9 B/s links, two subsets of 4 with a 50%
    cross-subset penalty (§5) -- reproduces the SPEC examples.
  * B200: MEASURED_PEAKS.json's sustained bf16 rate scaled by the measured GEMM
    efficiency of this repo, NVLink 5 through NVSwitch (900 GB/s per direction,
    one subset: every GPU reaches every peer at full rate), bf16 activations.
    `calibrate()` rescales the FLOP-derived phase times so the K=1 model
    equals a measured 1-GPU step (bench.py ms_per_step).
Pure analytical evaluation; deterministic; never times real execution.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field
from typing import Dict, List, Optional


@dataclass
class CostParams:
    flops_per_sec: float = 2e12          # per worker
    link_bandwidth: float = 6e9          # bytes/s per flow
    element_size: int = 4                # bytes per activation / gradient element
    cross_subset_penalty: float = 0.5    # throughput multiplier across subsets
    host_hop_latency: float = 10e-6      # seconds, cross-subset only (SPEC: arbitrary default)
    link_latency: float = 0.0            # seconds per transfer, any pair (B200: NCCL launch + NVSwitch hop)
    hbm_bandwidth: float = 0.0           # bytes/s for the FC weight streams and update (0: FLOPs only, as SPEC)
    fc_update_bytes: float = 18.0        # per FC parameter per step: fp32 w + momentum read/write, bf16 copy
    overlap_sync: bool = False           # B200 path: conv-gradient all-reduce overlaps conv backward
    sync_algorithm_factor: float = 1.0   # multiplier on 2(K-1)G/K (NVLS in-switch reduction ~0.5)

    def __post_init__(self):
        if min(self.flops_per_sec, self.link_bandwidth, self.element_size) <= 0:
            raise ValueError("CostParams: rates and element size must be positive")
        if not (0 < self.cross_subset_penalty <= 1):
            raise ValueError("CostParams: cross_subset_penalty must be in (0, 1]")


@dataclass
class Topology:
    K: int
    subsets: List[List[int]] = field(default_factory=list)

    def __post_init__(self):
        if not self.subsets:
            self.subsets = [list(range(self.K))]
        flat = sorted(w for s in self.subsets for w in s)
        if flat != list(range(self.K)):
            raise ValueError("Topology: subsets must partition 0..K-1")

    def same_subset(self, a: int, b: int) -> bool:
        return any(a in s and b in s for s in self.subsets)

    def all_same(self) -> bool:
        return len(self.subsets) == 1


PAPER = CostParams()


def paper_topology(K: int) -> Topology:
    """§5: GPUs with the same CPU parent (groups of 4) talk at full speed."""
    return Topology(K, [list(range(i, min(i + 4, K))) for i in range(0, K, 4)])


def b200_params(gemm_efficiency: float = 0.31, element_size: int = 2, hbm_efficiency: float = 0.75) -> CostParams:
    """NVLink 5 / NVSwitch: every GPU pair at 900 GB/s per direction (one subset),
    bf16 activations, the measured sustained bf16 rate x this repo's measured
    GEMM efficiency (bench.py roofline.frac). The FC layers are HBM-bound on
    B200 (tests/dev/cost_validate.py: 28% of the GEMM time for 7% of its
    FLOPs), so their time is max(FLOPs, weight bytes) at the measured copy
    bandwidth x the fused update's measured efficiency (fc6: 75%)."""
    return CostParams(flops_per_sec=1.406e15 * gemm_efficiency, link_bandwidth=900e9, element_size=element_size,
                      cross_subset_penalty=1.0, host_hop_latency=0.0, link_latency=10e-6, overlap_sync=True,
                      hbm_bandwidth=6.5456e12 * hbm_efficiency)


def b200_topology(K: int) -> Topology:
    return Topology(K)


# ---------------------------------------------------------------- primitives
def compute_time(flops: float, params: CostParams) -> float:
    if flops < 0:
        raise ValueError("compute_time: flops must be >= 0")
    return flops / params.flops_per_sec


def comm_time(nbytes: float, params: CostParams, same_subset: bool = True, concurrent_flows: int = 1) -> float:
    """bytes / (bandwidth * penalty if cross-subset) + latency if cross-subset;
    one sender's bandwidth is shared equally among its concurrent flows.
    link_latency (0 for the paper machine) is a per-transfer floor."""
    if nbytes < 0:
        raise ValueError("comm_time: bytes must be >= 0")
    bw = params.link_bandwidth / max(1, concurrent_flows)
    if same_subset:
        return nbytes / bw + params.link_latency
    return nbytes / (bw * params.cross_subset_penalty) + params.host_hop_latency + params.link_latency


def fc_matmul_balance(d: int, params: CostParams, K: int = 8) -> Dict[str, float]:
    """§5.1: per sample per worker, compute d*(d/K)*2 FLOPs vs receiving d
    elements (4096 x 4096 at K=8 is communication-bound)."""
    if d <= 0:
        raise ValueError("fc_matmul_balance: d must be positive")
    c = compute_time(d * (d / K) * 2, params)
    m = comm_time(d * params.element_size, params)
    return {"compute_s": c, "comm_s": m, "comm_bound": m > c}  # link_latency included for B200


# ---------------------------------------------------------------- model FLOPs
def model_flops(spec) -> Dict[str, object]:
    """Per-example GEMM FLOPs (2 per MAC): conv forward per layer, FC forward
    per layer (backward = 2x forward; conv1's dgrad is not computed)."""
    c, h, w = spec.input_shape
    conv = []
    for l in spec.conv_layers:
        def od(x):
            return (x + 2 * l.pad - l.kernel) // l.stride + 1
        oh, ow = od(h), od(w)
        conv.append(2.0 * oh * ow * l.out_channels * l.kernel * l.kernel * l.in_channels)
        h, w = oh, ow
        if l.pool_kernel:
            h, w = (h - l.pool_kernel) // l.pool_stride + 1, (w - l.pool_kernel) // l.pool_stride + 1
    fc = [2.0 * f.in_dim * f.out_dim for f in spec.fc_layers]
    return {"conv_fwd": conv, "fc_fwd": fc}



@dataclass
class Event:
    worker: int
    t0: float
    t1: float
    kind: str   # "compute" | "comm"
    label: str


@dataclass
class Timeline:
    """Events of worker 0 (workers are symmetric up to scheme B's root rotation).
    hidden_comm_fraction is over the scheme's boundary exchange (activations
    out, gradients back) -- the traffic the (b)/(c) pipelining hides; the
    model-parallel FC-internal collectives and the conv weight sync are
    reported separately (internal_s, sync_exposed_s)."""
    events: List[Event]
    step_time: float
    boundary_total: float = 0.0
    boundary_exposed: float = 0.0
    internal_s: float = 0.0
    sync_s: float = 0.0
    sync_exposed_s: float = 0.0

    @property
    def hidden_comm_fraction(self) -> Optional[float]:
        if self.boundary_total <= 0:
            return None
        return 1.0 - self.boundary_exposed / self.boundary_total

    def phase_table(self) -> Dict[str, float]:
        out: Dict[str, float] = {}
        for e in self.events:
            key = e.label.rstrip("0123456789")
            out[key] = out.get(key, 0.0) + (e.t1 - e.t0)
        return out

    def csv(self) -> str:
        rows = ["worker,t0,t1,kind,label"]
        rows += [f"{e.worker},{e.t0:.9e},{e.t1:.9e},{e.kind},{e.label}" for e in self.events]
        return "\n".join(rows) + "\n"


def exchange_elements(spec, K: int, b: int, scheme) -> Dict[str, float]:
    """Per-turn max-sender elements of the boundary exchange, the same counts
    cluster.cpp:502-528/615-673 charges (tests assert equality with
    step_accounting's trace): rows = examples one FC pass sees, turns = passes."""
    from .api import Scheme
    A = spec.flattened_conv_size()
    s = Scheme(int(scheme))
    if K == 1 or s == Scheme.DP:
        return {"turns": 1, "rows": b, "act": 0.0, "grad": 0.0, "act_flows": 0, "grad_flows": 0}
    if s == Scheme.A:   # all-gather: every worker ships its b rows to K-1 peers, partials come back the same way
        return {"turns": 1, "rows": K * b, "act": (K - 1) * b * A, "grad": (K - 1) * b * A,
                "act_flows": K - 1, "grad_flows": K - 1}
    if s == Scheme.B:   # root broadcasts b rows; every other worker returns its b x A partial to the root
        return {"turns": K, "rows": b, "act": (K - 1) * b * A, "grad": b * A, "act_flows": K - 1, "grad_flows": 1}
    q = b // K          # scheme C: every worker ships b/K rows to every peer, each way
    return {"turns": K, "rows": b, "act": (K - 1) * q * A, "grad": (K - 1) * q * A,
            "act_flows": K - 1, "grad_flows": K - 1}


def _flow_time(elems: float, flows: int, params: CostParams, topo: Topology) -> float:
    """Fan-out of `elems` over `flows` concurrent flows from one sender; the
    slowest (cross-subset when the topology has several subsets) bounds it."""
    if flows <= 0 or elems <= 0:
        return 0.0
    return comm_time(elems * params.element_size / flows, params, topo.all_same(), concurrent_flows=flows)


def scheme_step_model(spec, cluster, topo: Topology, params: CostParams,
                      compute_scale: float = 1.0) -> Timeline:
    """SPEC.md:442-452. Conv forward (data parallel) -> FC turns with the
    scheme's boundary exchange -> conv backward -> weight sync. Schemes B/C:
    exchange of turn j+1 runs while turn j computes (one turn of lookahead);
    gradient returns mirror it, so only the first exchange and the last return
    are exposed. Scheme A: gather, compute, scatter back-to-back.
    compute_scale multiplies every FLOP-derived compute time (calibration)."""
    from .api import Scheme
    K, b = cluster.workers, cluster.per_worker_batch
    s = Scheme(int(cluster.scheme))
    if K < 1 or b < 1 or (s == Scheme.C and K > 1 and b % K):
        raise ValueError("scheme_step_model: invalid workers/batch for the scheme")
    fl = model_flops(spec)
    ct = lambda f: compute_time(f, params) * compute_scale
    t_conv_f = ct(sum(fl["conv_fwd"]) * b)
    t_conv_b = ct((2 * sum(fl["conv_fwd"]) - fl["conv_fwd"][0]) * b)
    x = exchange_elements(spec, K, b, s)
    ev: List[Event] = [Event(0, 0.0, t_conv_f, "compute", "conv_fwd")]
    t = t_conv_f
    tl = Timeline(ev, 0.0)
    # FC weights this worker holds: the whole stack (K = 1, pure DP) or a 1/K
    # column shard; streamed twice per pass (fwd, dgrad; bf16) and updated once
    # per step when hbm_bandwidth is set
    P = sum(f.in_dim * f.out_dim for f in spec.fc_layers) / (1 if (K == 1 or s == Scheme.DP) else K)
    hbm = params.hbm_bandwidth
    fc_pass = lambda f: max(ct(f), 2 * 2 * P / hbm if hbm > 0 else 0.0)
    fc_upd = params.fc_update_bytes * P / hbm if hbm > 0 else 0.0
    if K == 1 or s == Scheme.DP:
        fc = fc_pass(3 * sum(fl["fc_fwd"]) * b)
        ev.append(Event(0, t, t + fc, "compute", "fc"))
        t += fc
    else:
        n = x["rows"]
        fc = fc_pass(3 * sum(fl["fc_fwd"]) * n / K)  # n examples over out/K columns
        # model-parallel internals per turn: forward all-gather of each layer's column
        # shard, backward reduce-scatter of the input partials above the first layer
        internal = sum(_flow_time((K - 1) * n * f.out_dim / K, K - 1, params, topo) for f in spec.fc_layers) + \
            sum(_flow_time((K - 1) * n * f.in_dim / K, K - 1, params, topo) for f in spec.fc_layers[1:])
        ta = _flow_time(x["act"], x["act_flows"], params, topo)
        tg = _flow_time(x["grad"], x["grad_flows"], params, topo)
        turn = fc + internal
        if s == Scheme.A:
            for lab, d, kind in (("exchange", ta, "comm"), ("fc", fc, "compute"),
                                 ("internal", internal, "comm"), ("return", tg, "comm")):
                ev.append(Event(0, t, t + d, kind, lab))
                t += d
            tl.boundary_total = tl.boundary_exposed = ta + tg
        else:
            link_out = t   # outbound exchange link free at
            starts = []
            for j in range(K):
                e0 = link_out if j == 0 else max(link_out, starts[-1])
                ev.append(Event(0, e0, e0 + ta, "comm", f"exchange{j}"))
                link_out = e0 + ta
                s0 = max(t, link_out)
                tl.boundary_exposed += s0 - t
                starts.append(s0)
                ev.append(Event(0, s0, s0 + fc, "compute", f"fc{j}"))
                ev.append(Event(0, s0 + fc, s0 + turn, "comm", f"internal{j}"))
                t = s0 + turn
            # returns travel opposite to the broadcasts and mirror them:
            # return j overlaps turn j+1, the last one is exposed
            link_back = 0.0
            for j in range(K):
                r0 = max(link_back, starts[j] + turn)
                ev.append(Event(0, r0, r0 + tg, "comm", f"return{j}"))
                link_back = r0 + tg
            tl.boundary_exposed += max(0.0, link_back - t)
            t = max(t, link_back)
            tl.boundary_total = K * (ta + tg)
        tl.internal_s = x["turns"] * internal
    if fc_upd > 0:
        ev.append(Event(0, t, t + fc_upd, "compute", "fc_update"))
        t += fc_upd
    ev.append(Event(0, t, t + t_conv_b, "compute", "conv_bwd"))
    t_end = t + t_conv_b
    if K > 1:
        G = sum(l.out_channels * l.in_channels * l.kernel ** 2 + l.out_channels for l in spec.conv_layers)
        if s == Scheme.DP:
            G += sum(f.in_dim * f.out_dim + f.out_dim for f in spec.fc_layers)
        sync_bytes = 2 * (K - 1) * G * 4 / K * params.sync_algorithm_factor  # SPEC.md:470, f32 gradients
        ts = comm_time(sync_bytes, params, topo.all_same()) + (len(spec.conv_layers) - 1) * params.link_latency
        # with overlap the per-layer all-reduce starts once the top layers' gradients are
        # final (DP: the FC gradients are final before conv backward starts)
        s0 = (t if s == Scheme.DP else t + 0.5 * t_conv_b) if params.overlap_sync else t_end
        ev.append(Event(0, s0, s0 + ts, "comm", "sync"))
        tl.sync_s, tl.sync_exposed_s = ts, max(0.0, s0 + ts - t_end)
        t_end = max(t_end, s0 + ts)
    tl.step_time = t_end
    return tl


def speedup(spec, cluster, topo: Topology, params: CostParams, compute_scale: float = 1.0) -> Dict[str, object]:
    """Images/s at K over images/s at K=1 with the same per-worker batch (weak scaling)."""
    one = dataclasses.replace(cluster, workers=1)
    t1 = scheme_step_model(spec, one, Topology(1), params, compute_scale).step_time
    tk = scheme_step_model(spec, cluster, topo, params, compute_scale)
    K = cluster.workers
    return {"step_time_1": t1, "step_time_K": tk.step_time, "speedup": K * t1 / tk.step_time,
            "images_per_s": K * cluster.per_worker_batch / tk.step_time,
            "hidden_comm_fraction": tk.hidden_comm_fraction, "timeline": tk}


def calibrate(spec, b: int, params: CostParams, measured_step_s: float) -> float:
    """compute_scale such that the K=1 model equals a measured 1-GPU step (the
    step time is non-decreasing in the scale; HBM-bound phases do not scale)."""
    from .api import ClusterConfig
    cl = ClusterConfig(workers=1, per_worker_batch=b)
    f = lambda sc: scheme_step_model(spec, cl, Topology(1), params, sc).step_time
    lo, hi = 0.0, 1.0
    while f(hi) < measured_step_s:
        hi *= 2.0
        if hi > 1e9:
            raise ValueError("calibrate: measured step unreachable")
    if f(lo) > measured_step_s:
        raise ValueError("calibrate: measured step below the model's memory-bound floor")
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        lo, hi = (mid, hi) if f(mid) < measured_step_s else (lo, mid)
    return 0.5 * (lo + hi)
