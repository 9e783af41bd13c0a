#!/usr/bin/env python
"""ASOT pairwise-distance benchmark (BASELINE.json metric) on 1..N B200s.

Default workload: c3 (BASELINE.json configs[2], the one it quotes "run at 1/2/4/8 GPUs", as the
metric is).  A step = the whole hot path over one batch: device-resident points,
offsets, weights, anchors and C_s  ->  mapping + histograms, Gibbs kernel, batched Sinkhorn on
every pair i < j, cost reduction  ->  the complete N x N matrix on rank 0.  Multi-GPU shards the
upper-triangular pair tiles (strong scaling of one fixed matrix) with the two NCCL exchanges of
distributed.py.  Timing: W untimed warm-up steps, then exactly K steps bracketed by barrier +
synchronize; each step is timed with CUDA events on the launch stream and the L2 is flushed
(256 MiB write) between steps outside the events; max over ranks.

Extra JSON keys: roofline (dominant kernel, live CUDA-event
timing via the library's profiling hook), cpu_baseline (the fp64 oracle on host cores, bounded
sample), e2e (host buffers through asot_distance_matrix_host), clocks, gpu_launches.
`--impl reference` times the oracle itself (this tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

TF32_OVER_BF16 = 1.1 / 2.25  # B200_PROFILING.md nominal dense tf32 / bf16
FP32_ALU_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # CUDA-core FFMA peak at max SM clock


DEBUG_ENV = ("ASOT_TC_DEBUG_MODE", "ASOT_PAIR_KERNEL", "ASOT_SOFT_DL_GENERIC", "ASOT_SPARSE")


def asot_env() -> dict:
    """Every ASOT_* environment variable of this run (recorded in the JSON line)."""
    return {k: v for k, v in sorted(os.environ.items()) if k.startswith("ASOT_")}


def cublas_tf32_tflops(dev) -> float:
    """Measured dense TF32 GEMM rate of this GPU through cuBLAS (torch.matmul 8192^3, TF32
    allowed; best of 3 x 5): context for the roofline denominator, which stays the
    MEASURED_PEAKS bf16 figure x the nominal tf32/bf16 ratio."""
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        n = 8192
        a = torch.randn(n, n, device=dev)
        b = torch.randn(n, n, device=dev)
        for _ in range(2):
            a @ b
        torch.cuda.synchronize()
        best = 0.0
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                a @ b
            e1.record()
            torch.cuda.synchronize()
            best = max(best, 5 * 2 * n ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
        del a, b
        return best
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def baseline_metric() -> str:
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        return json.load(f)["metric"]


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        d["_source"] = "measured"
        return d
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "_source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", str(self.gpu)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(self.NAMES, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def pairs_of(n: int) -> int:
    return n * (n - 1) // 2


# ------------------------------------------------------------------------------ oracle legs
def oracle_soft_map(inp, mapping, model, budget_s):
    """Soft-mapping oracle on the first distributions until ~budget_s; returns (H with those rows
    filled and the rest drawn from them, extrapolated full mapping seconds, description)."""
    from oracle import soft_oracle as S

    H = np.zeros((inp.n_dist, inp.n_anchors))
    t0 = time.perf_counter()
    done_pts = 0
    i = 0
    while i < inp.n_dist and (time.perf_counter() - t0) < budget_s:
        s, e = int(inp.offsets[i]), int(inp.offsets[i + 1])
        if mapping == "ml":
            Z, _ = S.ml_encode(inp.points[s:e], model.layers)
        else:
            Z, _, _ = S.dl_encode(inp.points[s:e], model.dictionary, model.lam_layers, model.n_layers)
        H[i] = S.soft_histograms(Z, inp.weights[s:e], np.array([0, e - s]))[0]
        done_pts += e - s
        i += 1
    t = time.perf_counter() - t0
    H[i:] = H[np.arange(inp.n_dist - i) % i]   # rows not mapped in the budget reuse mapped ones
    t_map = t / done_pts * inp.n_points
    return H, t_map, f"{mapping} encoder on {done_pts} points ({t:.2f} s), extrapolated to {inp.n_points}"


def oracle_sample_rate(inp, budget_s: float, seed: int = 0, mapping: str = "onehot", model=None):
    """The oracle (as it stands) on a bounded sample of the same workload: full mapping of every
    point (soft mappings: a timed sample of distributions, extrapolated), then Sinkhorn on seeded
    random pairs until the time budget.  Returns whole-job pairs/s extrapolated as
    P / (t_map + P / pair_rate), and a description."""
    from asot_inputs import random_pairs
    from oracle import asot_oracle as O

    if mapping == "onehot":
        # map whole distributions in order until half the budget; extrapolate by points
        H = np.zeros((inp.n_dist, inp.n_anchors))
        t0 = time.perf_counter()
        done_pts, i = 0, 0
        while i < inp.n_dist and (i < 2 or time.perf_counter() - t0 < budget_s / 2):
            s, e = int(inp.offsets[i]), int(inp.offsets[i + 1])
            _, h = O.map_and_histogram(inp.points[s:e], np.array([0, e - s]), inp.weights[s:e], inp.anchors)
            H[i] = h[0]
            done_pts += e - s
            i += 1
        t = time.perf_counter() - t0
        t_map = t / done_pts * inp.n_points
        H[i:] = H[np.arange(inp.n_dist - i) % i]   # rows not mapped in the budget reuse mapped ones
        map_note = (f"one-hot mapping of {i} distributions / {done_pts} points ({t:.2f} s), extrapolated "
                    f"to all {inp.n_points} points")
    else:
        H, t_map, map_note = oracle_soft_map(inp, mapping, model, budget_s / 2)
    cost = inp.cost
    if mapping == "ml":
        from oracle import soft_oracle as S
        t0 = time.perf_counter()
        cost = S.mahalanobis_cost(inp.anchors, model.M, normalize=True)
        t_map += time.perf_counter() - t0
    pi, pj = random_pairs(inp.n_dist, 200000, seed=seed)
    done, t_pairs, batch = 0, 0.0, 256
    while t_pairs < budget_s and done < len(pi):
        s = time.perf_counter()
        O.pair_costs(H, cost, inp.eps, inp.iters, pi[done:done + batch].astype(np.int64),
                     pj[done:done + batch].astype(np.int64), batch=batch)
        t_pairs += time.perf_counter() - s
        done += len(pi[done:done + batch])
    rate = done / t_pairs
    P = inp.n_pairs
    value = P / (t_map + P / rate)
    sample = (f"fp64 oracle: {map_note} + Sinkhorn on "
              f"{done} seeded random pairs ({t_pairs:.2f} s, {rate:.0f} pairs/s); whole-job "
              f"throughput extrapolated to all {P} pairs")
    return value, sample


def run_reference(args, inp, rank, world):
    """--impl reference: the oracle as it stands, each step a bounded sample of the workload.

    Same metric as our arm -- whole-job pairs/s for the N x N matrix -- extrapolated the same
    way as cpu_baseline: each step maps a seeded sample of distributions (mapping time per point
    -> all points) and runs the fp64 Sinkhorn on a seeded sample of pairs among them (time per
    pair -> all P pairs); value = P / (t_map_all + P * t_pair) over the pooled timings."""
    if rank != 0:
        return
    from oracle import asot_oracle as O

    cores = len(os.sched_getaffinity(0))
    m = max(2, args.ref_dists)
    n_sample = args.ref_pairs

    def ref_step(k):
        rng = np.random.default_rng(1000 + k)
        dists = np.sort(rng.choice(inp.n_dist, size=min(m, inp.n_dist), replace=False))
        H = np.zeros((inp.n_dist, inp.n_anchors))
        t0 = time.perf_counter()
        pts = 0
        for d in dists:
            s, e = int(inp.offsets[d]), int(inp.offsets[d + 1])
            _, h = O.map_and_histogram(inp.points[s:e], np.array([0, e - s]), inp.weights[s:e],
                                       inp.anchors)
            H[d] = h[0]
            pts += e - s
        t_map = time.perf_counter() - t0
        iu, ju = np.triu_indices(len(dists), k=1)
        sel = rng.choice(len(iu), size=min(n_sample, len(iu)), replace=False)
        pi, pj = dists[iu[sel]].astype(np.int64), dists[ju[sel]].astype(np.int64)
        t0 = time.perf_counter()
        O.pair_costs(H, inp.cost, inp.eps, inp.iters, pi, pj)
        return t_map, pts, time.perf_counter() - t0, len(pi)

    for k in range(args.warmup):
        ref_step(-1 - k)
    tm = tp = 0.0
    npts = npairs = 0
    t0 = time.perf_counter()
    for k in range(args.steps):
        a, b, c, d = ref_step(k)
        tm, npts, tp, npairs = tm + a, npts + b, tp + c, npairs + d
    dt = time.perf_counter() - t0
    P = inp.n_pairs
    value = P / (tm / npts * inp.n_points + P * tp / npairs)
    sample = (f"per step: mapping of {m} seeded distributions + fp64 Sinkhorn (L={inp.iters}) on "
              f"{min(n_sample, m * (m - 1) // 2)} seeded pairs among them; whole-job pairs/s "
              f"extrapolated from the pooled times ({npts} points mapped in {tm:.2f} s, {npairs} "
              f"pairs in {tp:.2f} s) to all {inp.n_points} points and {P} pairs")
    line = {
        "impl": "reference", "metric": baseline_metric(), "value": value, "unit": "pairs/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(inp, args, world),
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": cores, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(inp, args, world):
    return {
        "workload": f"{inp.name} (BASELINE.json configs[{int(inp.name[1]) - 1}]): N={inp.n_dist} "
                    f"distributions, K={inp.n_anchors} anchors, d={inp.dim}, L={inp.iters}, "
                    f"eps={float(inp.eps)}" + (" -- the config BASELINE.json runs at 1/2/4/8 GPUs, "
                                               "as the metric is quoted" if inp.name == "c3" else ""),
        "n_dist": inp.n_dist, "n_points": inp.n_points, "dim": inp.dim,
        "n_anchors": inp.n_anchors, "iters": inp.iters, "pairs": inp.n_pairs,
        "precision": args.precision, "l2_flush": "256 MiB write between timed steps",
        "parallelism": f"pair-tiles x{world}",
        "mapping": getattr(args, "mapping", "onehot"),
        "anchors": (getattr(args, "anchors", "seeded") if getattr(args, "anchors", "seeded") == "seeded"
                    else f"kmeans (iters={args.kmeans_iters}, batch={args.kmeans_batch}, in every step)"),
    }


# ------------------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # default: configs[2] (c3), the config BASELINE.json quotes "at 1/2/4/8 GPUs" like the metric
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--precision", default="tf32", choices=["tf32", "fp32"])
    ap.add_argument("--anchors", default="seeded", choices=["seeded", "kmeans"],
                    help="seeded anchors (the north-star path) or NEXT-2 ASOT-k: anchors learned "
                         "inside every step by mini-batch k-means (Forgy init + batch draws seeded)")
    ap.add_argument("--kmeans-iters", type=int, default=50)
    ap.add_argument("--kmeans-batch", type=int, default=4096)
    ap.add_argument("--baseline", default="none", choices=["none", "eot"],
                    help="NEXT-4: also time entropic OT on the original point sets (the paper's "
                         "eOT / BDS-eOT comparison) on a seeded pair sample, on the same GPU")
    ap.add_argument("--eot-pairs", type=int, default=20000)
    ap.add_argument("--exact", action="store_true",
                    help="NEXT-3: also solve exact anchor-space OT on a seeded pair sample and report "
                         "its pairs/s and the eASOT-vs-exact gap")
    ap.add_argument("--exact-pairs", type=int, default=0, help="exact-ASOT sample (0: 20000, 1000 if K > 128)")
    ap.add_argument("--bounds", action="store_true",
                    help="NEXT-3: Prop. 1 / Prop. 2 bound terms, exact W_AS and exact W_1 on the original "
                         "points (Euclidean metric) on a pair sample, with violation counts")
    ap.add_argument("--bounds-pairs", type=int, default=20000)
    ap.add_argument("--pairs-api", action="store_true",
                    help="also time asot_pairwise_sinkhorn (SPEC batched_sinkhorn_fixed) on the whole "
                         "upper triangle given as an explicit (shuffled) pair list")
    ap.add_argument("--mapping", default="onehot", choices=["onehot", "ml", "dl"],
                    help="P: one-hot nearest anchor (the north-star path), or the NEXT-1 soft "
                         "mappings ASOT-ML / ASOT-DL (seeded parameters)")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--ref-pairs", type=int, default=256)
    ap.add_argument("--ref-dists", type=int, default=24, help="distributions mapped per reference step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--n-dist", type=int, default=None,
                    help="shrink N (profiling runs only; bench lines use the full config)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    # diagnostic kernel selection must never reach a bench line: the
    # epilogue/MMA-skipping variants exist only in ASOT_DEBUG_BUILD libraries, and the
    # cross-check kernel switches are for tests
    bad_env = [k for k in DEBUG_ENV if os.environ.get(k)]
    if bad_env:
        raise SystemExit(f"bench.py refuses to run with diagnostic kernel selection set: {bad_env}")

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    from asot_inputs import make_inputs

    inp = make_inputs(args.config, n_dist=args.n_dist)
    soft_model = None
    if args.mapping == "ml":
        from asot_inputs.soft import make_ml_model
        soft_model = make_ml_model(inp.dim, inp.n_anchors)
    elif args.mapping == "dl":
        from asot_inputs.soft import make_dl_inputs
        inp, soft_model = make_dl_inputs(args.config, n_dist=args.n_dist)
    if args.impl == "reference":
        run_reference(args, inp, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_2310_16123_b200 as asot
    from paper_2310_16123_b200 import distributed as D_

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    prec = asot.TF32 if args.precision == "tf32" else asot.FP32
    eff = asot.effective_precision(inp.n_anchors, prec)

    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    pts, offs, w, anc, cst = t(inp.points), t(inp.offsets), t(inp.weights), t(inp.anchors), t(inp.cost)
    cmax = float(inp.cost.max())
    status = asot.asot.new_status(dev)
    ws = asot.Workspace(dev)
    Dbuf = torch.empty((inp.n_dist, inp.n_dist), dtype=torch.float32, device=dev)
    n_tiles = asot.num_tiles(inp.n_dist)
    launches = [0]

    exchange_note = ["single GPU: no exchange"]
    last_H, last_A = [None], [None]   # the histograms / learned anchors of the last step (path kind)
    if (args.mapping != "onehot" or args.anchors != "seeded") and world > 1:
        raise SystemExit("--mapping ml/dl and --anchors kmeans are single-GPU in this build")
    km_events = []
    if args.anchors == "kmeans":
        if args.mapping != "onehot":
            raise SystemExit("--anchors kmeans runs with the one-hot mapping (ASOT-k)")
        from asot_inputs.soft import make_kmeans_draws
        km_init, km_idx = make_kmeans_draws(inp.points, inp.n_anchors, args.kmeans_iters,
                                            args.kmeans_batch)
        km_init_d, km_idx_d = t(km_init), t(km_idx)
    if args.mapping == "ml":
        m = soft_model
        mW1, mb1, mW2, mb2, mM = t(m.W1), t(m.b1), t(m.W2), t(m.b2), t(m.M)

        def step():
            H, _, _ = asot.map_soft_ml(pts, offs, w, mW1, mb1, mW2, mb2, offsets_host=inp.offsets,
                                       status=status)
            last_H[0] = H
            launches[0] += asot.last_launch_count()
            C = asot.mahalanobis_cost(anc, mM, normalize=True, workspace=ws)
            launches[0] += 3
            asot.distance_matrix(None, None, None, None, C, float(inp.eps), inp.iters,
                                 precision=prec, hist=H, out=Dbuf, cost_max=1.0, status=status,
                                 workspace=ws)
            launches[0] += asot.last_launch_count()
            return Dbuf
    elif args.mapping == "dl":
        m = soft_model
        dV1, dc1, dv2, dc2 = t(m.V1), t(m.c1), t(m.v2.reshape(-1)), t(m.c2)

        def step():
            H, _, _ = asot.map_soft_dl(pts, offs, w, anc, dV1, dc1, dv2, dc2, m.n_layers,
                                       offsets_host=inp.offsets, status=status)
            last_H[0] = H
            launches[0] += asot.last_launch_count()
            asot.distance_matrix(None, None, None, None, cst, float(inp.eps), inp.iters,
                                 precision=prec, hist=H, out=Dbuf, cost_max=cmax, status=status,
                                 workspace=ws)
            launches[0] += asot.last_launch_count()
            return Dbuf
    elif args.anchors == "kmeans":
        def step():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _, A, _, _ = asot.kmeans_minibatch(pts, km_init_d, km_idx_d, status=status)
            last_A[0] = A
            e1.record()
            km_events.append((e0, e1))
            launches[0] += asot.last_launch_count()
            C = asot.sqeuclid_cost(A)
            launches[0] += 2
            asot.distance_matrix(pts, offs, w, A, C, float(inp.eps), inp.iters, precision=prec,
                                 out=Dbuf, offsets_host=inp.offsets, cost_max=1.0, status=status,
                                 workspace=ws)
            launches[0] += asot.last_launch_count()
            return Dbuf
    elif world == 1:
        def step():
            asot.distance_matrix(pts, offs, w, anc, cst, float(inp.eps), inp.iters, precision=prec,
                                 out=Dbuf, offsets_host=inp.offsets, cost_max=cmax, status=status,
                                 workspace=ws)
            launches[0] += asot.last_launch_count()
            return Dbuf
    else:
        steps_impl = D_.cuda_steps(pts, offs, inp.offsets, w, anc, cst, float(inp.eps), inp.iters,
                                   prec, cmax, status, workspace=ws)

        def counted(fn):
            def inner(*a):
                r = fn(*a)
                launches[0] += asot.last_launch_count()
                return r
            return inner

        steps_impl = D_.DistSteps(counted(steps_impl.map_range), counted(steps_impl.tiles),
                                  counted(steps_impl.unpack), counted(steps_impl.zero_diag),
                                  counted(steps_impl.tiles_into), counted(steps_impl.map_range_bcast))
        # result exchange: NVLink stores from the Sinkhorn epilogue into rank 0's symmetric-memory
        # matrix (one kernel does compute + "gather"); NCCL all-gather + unpack as the fallback
        p2p = None
        if os.environ.get("ASOT_RESULT_EXCHANGE", "p2p") == "p2p":
            try:
                p2p = D_.P2PResult(inp.n_dist, dev, n_anchors=inp.n_anchors)
                exchange_note[0] = ("p2p: histogram rows stored into every rank's symmetric-memory H, "
                                    "distances stored into rank 0's symmetric-memory matrix (NVLink)")
            except Exception as exc:  # noqa: BLE001 - report and fall back
                exchange_note[0] = f"nccl all-gather + unpack (symmetric memory unavailable: {exc!s:.80})"
            # every rank must take the same exchange: fall back everywhere if any rank failed
            ok = torch.tensor([1 if p2p is not None else 0], dtype=torch.int32, device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if int(ok.item()) == 0 and p2p is not None:
                p2p = None
                exchange_note[0] = "nccl all-gather + unpack (symmetric memory unavailable on a peer rank)"

        def step():
            if p2p is not None:
                return D_.distance_matrix_distributed_p2p(inp.n_dist, inp.n_anchors, inp.offsets,
                                                          n_tiles, steps_impl, p2p, device=dev)
            return D_.distance_matrix_distributed(inp.n_dist, inp.n_anchors, inp.offsets, n_tiles,
                                                  steps_impl, device=dev)

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    asot.check_status(status)

    def timed_region():
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        asot.asot.profile_enable(True)
        asot.asot.profile_read(reset=True)
        asot.asot.profile_read(reset=True, kernel=asot.asot.PROF_MAP)
        launches[0] = 0
        clocks = ClockSampler(local_rank if "CUDA_VISIBLE_DEVICES" not in os.environ else 0)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clocks.start()
        time.sleep(0.2)
        wall0 = time.perf_counter()
        Dres = None
        for k in range(args.steps):
            flush.zero_()
            evs[k][0].record(stream)
            torch.cuda.nvtx.range_push(f"asot step {k}")
            Dres = step()
            torch.cuda.nvtx.range_pop()
            evs[k][1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        wall = time.perf_counter() - wall0
        clk = clocks.stop()
        asot.asot.profile_enable(False)
        kern_ms, kern_n = asot.asot.profile_read(reset=True)
        map_ms, map_n = asot.asot.profile_read(reset=True, kernel=asot.asot.PROF_MAP)
        step_ms = [a.elapsed_time(b) for a, b in evs]
        return Dres, wall, clk, kern_ms, kern_n, map_ms, map_n, step_ms, launches[0]

    # a timed region that saw hardware / thermal slowdown is rejected and re-measured once
    # (sw_power_cap is kept and reported)
    BAD = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    Dres, wall, clk, kern_ms, kern_n, map_ms, map_n, step_ms, gpu_launches = timed_region()
    bad = torch.tensor([1 if BAD & set(clk.get("reasons") or []) else 0], dtype=torch.int64,
                       device=dev)
    if world > 1:
        dist.all_reduce(bad, op=dist.ReduceOp.MAX)
    if int(bad.item()):
        first_reasons = clk.get("reasons")
        Dres, wall, clk, kern_ms, kern_n, map_ms, map_n, step_ms, gpu_launches = timed_region()
        clk["remeasured_after"] = first_reasons
    tot_ms = sum(step_ms)
    if world > 1:
        tt = torch.tensor([tot_ms, kern_ms / max(kern_n, 1)], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        tot_ms, kern_avg_ms = float(tt[0]), float(tt[1])
        gl = torch.tensor([gpu_launches], dtype=torch.int64, device=dev)
        dist.all_reduce(gl)
        gpu_launches = int(gl.item())
    else:
        kern_avg_ms = kern_ms / max(kern_n, 1)
    asot.check_status(status)
    if rank == 0:
        Dh = Dres
        assert torch.isfinite(Dh).all() and torch.equal(Dh, Dh.T) and torch.all(torch.diagonal(Dh) == 0)

    P = inp.n_pairs
    value = P * args.steps / (tot_ms / 1e3)

    # ---- roofline of the dominant kernel (Sinkhorn, a5+a6), live CUDA-event timing
    K, L = inp.n_anchors, inp.iters
    flops_per_pair = 4 * K * K * L + 2 * K * K           # SURVEY §8(d) algorithmic work per pair
    pairs_per_launch = P if world == 1 else -(-P // world)
    peaks = measured_peaks()
    # which Sinkhorn kernel the calls ran: the library decides on the device from the histograms'
    # supports (asot_sinkhorn_path_kind states the rule); recompute them here for the report
    if last_H[0] is not None:
        H_path = last_H[0]
    else:
        _, H_path, _ = asot.map_to_anchors(pts, offs, w, last_A[0] if last_A[0] is not None else anc,
                                           offsets_host=inp.offsets)
    supports = (H_path != 0).sum(dim=1).to(torch.float64)
    kind = asot.asot.sinkhorn_path_kind(H_path, prec)
    # hardware MAC rate of the kernel's MMA kind (per SM per clock) and MMAs per algorithmic product
    mac_clk, per_product = {10: (4096, 3), 3: (2048, 3), 5: (2048, 3)}.get(kind, (2048, 1))
    sparse_info = None
    if kind == 11:
        # the small-support kernels (R#36): thread per pair, an S x S register block of K per
        # support class (S = 4, 6, 8; 9-16 bins: a half-warp per pair), fp32 FFMA2 -- bound by the
        # FP32 pipe / issue rate.  Issued work: 2 updates x S^2 MACs per iteration; useful work:
        # the real |S_a| x |S_b| blocks (sum over i < j of m_i m_j)
        S = supports
        useful_mn = float((S.sum() ** 2 - (S * S).sum()) / 2) if world == 1 else None
        # issued: the register form each pair runs (support-ordered classes, pair (i', j'), i' < j':
        # the R x C rectangle R = class of supp(i'), C = class of supp(j') for C in {4, 6, 8}, the
        # 16 x 16 half-warp form when C = 16): sum over pairs of 4 R C L
        ss = np.sort(S.cpu().numpy())
        form = np.where(ss <= 4, 4, np.where(ss <= 6, 6, np.where(ss <= 8, 8, 16))).astype(np.float64)
        rows_before = np.concatenate([[0.0], np.cumsum(form)[:-1]])   # sum of R over i' < j'
        per_col = np.where(form == 16, 256.0 * np.arange(ss.size), form * rows_before)
        flops_issued = float((4.0 * L * per_col).sum() / max(P, 1))
        peak = FP32_ALU_PEAK_TFLOPS
        bound, peak_note = "alu", "FP32 FFMA: 148 SMs x 128 lanes x 2 x 1.965 GHz"
        sparse_info = {"max_support": int(S.max()), "mean_support": float(S.mean()),
                       "issued_flops_per_pair_mean": flops_issued,
                       "useful_flops_per_pair_mean": (4 * L + 2) * useful_mn / P if useful_mn else None,
                       "dense_equivalent_flops_per_pair": flops_per_pair}
        flops_per_pair = flops_issued
    elif kind == 10:
        peak = peaks["bf16_tflops"] / 3
        bound, peak_note = "tensor", (f"BF16x3: dense BF16 ({peaks['_source']} {peaks['bf16_tflops']} TFLOP/s "
                                      f"burst) / 3 MMAs per algorithmic product")
    elif kind in (3, 5):
        peak = peaks["bf16_tflops"] * TF32_OVER_BF16 / 3
        bound, peak_note = "tensor", (f"3xTF32: dense TF32 ({peaks['_source']} bf16 {peaks['bf16_tflops']} "
                                      f"TFLOP/s burst x 1.1/2.25) / 3 MMAs per algorithmic product")
    elif eff == asot.TF32:
        peak = peaks["bf16_tflops"] * TF32_OVER_BF16
        bound, peak_note = "tensor", (f"dense TF32 = {peaks['_source']} bf16 {peaks['bf16_tflops']} "
                                      f"TFLOP/s (burst) x nominal tf32/bf16 1.1/2.25")
    else:
        peak = FP32_ALU_PEAK_TFLOPS
        bound, peak_note = "alu", "FP32 FFMA: 148 SMs x 128 lanes x 2 x 1.965 GHz"
    achieved = flops_per_pair * pairs_per_launch / (kern_avg_ms / 1e3) / 1e12
    # ncu evidence for this kernel and workload (profiles/ncu_summary.json, written from the
    # committed `ncu --set full` captures by tools/summarize_ncu.py: a run under ncu is never
    # the bench run, so these are the capture's per-launch numbers, named with their source)
    traffic, ncu_ev = None, None
    spath = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(spath):
        with open(spath) as f:
            ncu_ev = json.load(f).get(f"{inp.name}:{args.precision}")
        if kind == 11:
            with open(spath) as f:
                ncu_ev = json.load(f).get(f"{inp.name}:sparse")
        if ncu_ev:
            traffic = ncu_ev.get("dram_bytes_per_launch")
    roofline = {"bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": asot.asot.KERNEL_NAMES[kind],
                "kernel_ms_per_launch": kern_avg_ms,
                "kernel_share_of_step": kern_avg_ms * kern_n / max(tot_ms, 1e-9) if world == 1 else None,
                "flops_per_pair": flops_per_pair, "pairs_per_launch": pairs_per_launch,
                "peak_note": peak_note,
                "peak_sustained_based": peaks.get("bf16_tflops_sustained", 0) * (TF32_OVER_BF16 if eff == asot.TF32 else 0) or None,
                "ncu": ncu_ev}
    if sparse_info is not None:
        sparse_info["useful_tflops"] = (sparse_info["useful_flops_per_pair_mean"] or 0) * pairs_per_launch / (kern_avg_ms / 1e3) / 1e12
        sparse_info["useful_frac"] = sparse_info["useful_tflops"] / peak
        roofline["sparse"] = sparse_info
        roofline["kernel_ms_note"] = ("the timed Sinkhorn launch scope = support extraction + fp32 K images "
                                      "(sparse prep) + the small-support kernel + the dense kernel's "
                                      "immediate return")
    if bound == "tensor" and rank == 0:
        ct = cublas_tf32_tflops(dev)
        roofline["cublas_tf32_measured_tflops"] = ct
        roofline["frac_of_cublas_tf32"] = achieved / (ct / (3 if kind in (3, 5) else 1)) if kind != 10 else None
    if bound == "tensor":
        # context: the hardware's nominal dense TF32 rate (2048 MAC/clk/SM, tools/cg2_rate.cu) at the
        # median SM clock sampled during the timed region (3xTF32: one third of it)
        mhz = (clk or {}).get("sm_mhz") or 1965.0
        nominal = mac_clk * 2 * 148 * mhz * 1e6 / 1e12 / per_product
        roofline["nominal_peak_at_clock"] = nominal
        roofline["frac_of_nominal"] = achieved / nominal
        # the clock the last timed launch actually ran at (in-kernel %clock64 / %globaltimer
        # probe; under power capping it sits below the clock nvidia-smi reports)
        try:
            emhz = asot.asot.profile_clock(kind)
        except Exception:  # noqa: BLE001 -- kind without a probe
            emhz = None
        if emhz:
            enominal = mac_clk * 2 * 148 * emhz * 1e6 / 1e12 / per_product
            roofline["effective_sm_mhz"] = emhz
            roofline["nominal_peak_at_effective_clock"] = enominal
            roofline["frac_of_nominal_effective"] = achieved / enominal

    # ---- mapping step (a2): the north star's "achieved HBM GB/s for mapping", next to the
    # FP32-pipe fraction that actually bounds it; live CUDA-event timing
    mapping = None
    if map_n:
        map_avg_ms = map_ms / map_n
        T_rank = inp.n_points if world == 1 else None
        if T_rank is not None and args.mapping != "onehot":
            d_, K_ = inp.dim, inp.n_anchors
            if args.mapping == "ml":
                h_ = 2 * d_
                flops_pt = 2 * d_ * h_ + 2 * h_ * K_
                kname = "soft_map_kernel<ML> (MLP d->2d->K, |.|/l1, fused a' = Z^T a)"
            else:
                h_ = max(1, d_ // 2)
                flops_pt = 2 * d_ * h_ + 2 * h_ + soft_model.n_layers * 4 * d_ * K_
                kname = f"soft_map_kernel<DL> ({soft_model.n_layers} near-one-hot layers, fused a' = Z^T a)"
            bytes_ = T_rank * (4 * d_ + 4) + inp.n_dist * K_ * 4
            dl_tc = (args.mapping == "dl" and not os.environ.get("ASOT_SOFT_DL_GENERIC")
                     and asot.asot._lib_handle().asot_map_soft_dl_workspace_bytes(d_, K_, T_rank) > 0)
            if dl_tc:
                # g = W^T r on the tensor cores: 3 TF32 MMAs per product (3xTF32), the sparse r
                # gather and the lambda MLP on the CUDA cores (asot_soft_dl_tc.cu)
                L_ = soft_model.n_layers
                g_flops = L_ * 2 * d_ * K_ * T_rank
                tpeak = peaks["bf16_tflops"] * TF32_OVER_BF16
                mapping = {
                    "kernel": f"soft_dl_tc_kernel ({L_} near-one-hot layers; g = W^T r on tcgen05 3xTF32, "
                              "sparse r = W z - x gather)",
                    "ms_per_launch": map_avg_ms, "points_per_launch": T_rank,
                    "g_flops_per_point": L_ * 2 * d_ * K_,
                    "bound": "tensor",
                    "g_tflops_algorithmic": g_flops / (map_avg_ms / 1e3) / 1e12,
                    "tf32_issued_tflops": 3 * g_flops / (map_avg_ms / 1e3) / 1e12,
                    "tf32_peak_tflops": tpeak,
                    "tf32_frac": 3 * g_flops / (map_avg_ms / 1e3) / 1e12 / tpeak,
                    "hbm_gbs": bytes_ / (map_avg_ms / 1e3) / 1e9, "hbm_peak_gbs": peaks.get("hbm_gbs"),
                    "share_of_step": map_ms / max(tot_ms, 1e-9),
                    "note": "tf32_frac counts the three TF32 MMAs per product against dense TF32 "
                            "(measured bf16 x 1.1/2.25); the r gather between layers leaves the "
                            "tensor pipe idle (DESIGN.md, DL TC kernel)"}
            ml_tc = (args.mapping == "ml"
                     and asot.asot._lib_handle().asot_map_soft_ml_workspace_bytes(d_, h_, K_) > 0)
            if ml_tc:
                # both MLP layers on the tensor cores: 3 BF16 MMAs per product (BF16x3 split,
                # asot_soft_ml_tc.cu), against the measured dense BF16 peak
                flops = flops_pt * T_rank
                bpeak = peaks["bf16_tflops"]
                mapping = {
                    "kernel": "soft_ml_tc_kernel (MLP d->2d->K on tcgen05 kind::f16, BF16x3 split; "
                              "|.|/l1 and fp64 a' = Z^T a on the CUDA cores)",
                    "ms_per_launch": map_avg_ms, "points_per_launch": T_rank,
                    "flops_per_point": flops_pt, "bound": "tensor",
                    "tflops_algorithmic": flops / (map_avg_ms / 1e3) / 1e12,
                    "bf16_issued_tflops": 3 * flops / (map_avg_ms / 1e3) / 1e12,
                    "bf16_peak_tflops": bpeak,
                    "bf16_frac": 3 * flops / (map_avg_ms / 1e3) / 1e12 / bpeak,
                    "hbm_gbs": bytes_ / (map_avg_ms / 1e3) / 1e9, "hbm_peak_gbs": peaks.get("hbm_gbs"),
                    "share_of_step": map_ms / max(tot_ms, 1e-9),
                    "note": "bf16_frac counts the three BF16 MMAs per product; per 128-point tile the "
                            "layers run back to back (relu/split epilogue between them) and a CUDA-core "
                            "pass normalises the codes and sums the histogram"}
        if T_rank is not None and args.mapping != "onehot" and mapping is None:
            mapping = {
                "kernel": kname, "ms_per_launch": map_avg_ms, "points_per_launch": T_rank,
                "flops_per_point": flops_pt,
                "fp32_tflops": flops_pt * T_rank / (map_avg_ms / 1e3) / 1e12,
                "fp32_peak_tflops": FP32_ALU_PEAK_TFLOPS,
                "fp32_frac": flops_pt * T_rank / (map_avg_ms / 1e3) / 1e12 / FP32_ALU_PEAK_TFLOPS,
                "hbm_gbs": bytes_ / (map_avg_ms / 1e3) / 1e9, "hbm_peak_gbs": peaks.get("hbm_gbs"),
                "share_of_step": map_ms / max(tot_ms, 1e-9),
                "note": "CUDA-core fp32 GEMM-like tiles (16 points x weights from L2/SMEM); "
                        "bound: FP32 FFMA peak 148 x 128 x 2 x 1.965 GHz"}
        elif T_rank is not None and args.mapping == "onehot" and inp.dim in (32, 64, 128) and \
                inp.n_anchors % 64 == 0 and world == 1:
            # asot_distance_matrix maps on the tensor cores (R#37: asot_map_tc.cu's rule, d in
            # {32, 64, 128}, K % 64 == 0) + the exact kernel on the listed ambiguous points
            d_, K_ = inp.dim, inp.n_anchors
            bytes_ = T_rank * (4 * d_ + 4) + K_ * d_ * 4
            flops = 2 * K_ * d_ * T_rank                      # x . w per (point, anchor)
            tpeak = peaks["bf16_tflops"] * TF32_OVER_BF16
            mapping = {
                "kernel": "map_tc_kernel (tcgen05 3xTF32 scores, R#37 bound) + map_assign_kernel on the "
                          "ambiguous points", "ms_per_launch": map_avg_ms, "points_per_launch": T_rank,
                "bound": "tensor", "hbm_gbs": bytes_ / (map_avg_ms / 1e3) / 1e9,
                "hbm_peak_gbs": peaks.get("hbm_gbs"),
                "hbm_frac": bytes_ / (map_avg_ms / 1e3) / 1e9 / peaks.get("hbm_gbs", 6650.0),
                "tflops_algorithmic": flops / (map_avg_ms / 1e3) / 1e12,
                "tf32_issued_frac": 3 * flops / (map_avg_ms / 1e3) / 1e12 / tpeak,
                "share_of_step": map_ms / max(tot_ms, 1e-9),
                "note": "ms covers the norms / images prep, the tensor-core pass and the exact pass on "
                        "the listed points; the decision is the fp64 definition's (bit-exact tests)"}
        elif T_rank is not None and args.mapping == "onehot":
            d_, K_ = inp.dim, inp.n_anchors
            bytes_ = T_rank * (4 * d_ + 4) + K_ * d_ * 4     # points in, assignment out, anchors
            lane_ops = 2 * K_ * d_ * T_rank                   # FSUB + FFMA per (point, anchor, dim)
            mapping = {
                "kernel": "map_assign_kernel", "ms_per_launch": map_avg_ms,
                "points_per_launch": T_rank,
                "hbm_gbs": bytes_ / (map_avg_ms / 1e3) / 1e9, "hbm_peak_gbs": peaks.get("hbm_gbs"),
                "hbm_frac": bytes_ / (map_avg_ms / 1e3) / 1e9 / peaks.get("hbm_gbs", 6650.0),
                "fp32_tflops": 3 * K_ * d_ * T_rank / (map_avg_ms / 1e3) / 1e12,
                "fp32_pipe_frac": lane_ops / (map_avg_ms / 1e3) / (FP32_ALU_PEAK_TFLOPS / 2 * 1e12),
                "share_of_step": map_ms / max(tot_ms, 1e-9),
                "note": "ALU-bound by design (intensity 3Kd/(4d+8) >> FP32 ridge); fp32_pipe_frac = "
                        "2Kd lane-ops per point / (148 SMs x 128 lanes x 1.965 GHz)"}

    kmeans = None
    if km_events:
        timed = km_events[-args.steps:]
        km_ms = sum(a.elapsed_time(b) for a, b in timed) / len(timed)
        pts_assigned = args.kmeans_iters * args.kmeans_batch
        kmeans = {"iters": args.kmeans_iters, "batch": args.kmeans_batch, "ms_per_step": km_ms,
                  "points_assigned_per_s": pts_assigned / (km_ms / 1e3),
                  "launches_per_step": 1 + 2 * args.kmeans_iters,
                  "share_of_step": km_ms * len(timed) / max(tot_ms, 1e-9),
                  "note": "per iteration: map_assign_kernel on the gathered batch + one update "
                          "launch (K CTAs); launch-latency bound at these batch sizes"}

    # ---- NEXT-4: the paper's comparison system on the same box (eOT on the original points)
    eot_base = None
    if args.baseline == "eot" and rank == 0:
        from asot_inputs import anchor_sqdist_scale, random_pairs
        scale = float(anchor_sqdist_scale(inp.anchors))
        ei, ej = random_pairs(inp.n_dist, min(args.eot_pairs, inp.n_pairs), seed=77)
        ei_d, ej_d = t(ei.astype(np.int32)), t(ej.astype(np.int32))
        est = asot.asot.new_status(dev)
        asot.eot_pairs(pts, offs, w, ei_d, ej_d, float(inp.eps), inp.iters, scale,
                       offsets_host=inp.offsets, status=est)          # warm-up
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d_eot = asot.eot_pairs(pts, offs, w, ei_d, ej_d, float(inp.eps), inp.iters, scale,
                               offsets_host=inp.offsets, status=est)
        e1.record()
        torch.cuda.synchronize()
        asot.check_status(est)
        ms = e0.elapsed_time(e1)
        de = d_eot.cpu().numpy().astype(np.float64)
        da = Dres.cpu().numpy()[ei, ej].astype(np.float64) if world == 1 else None
        rate = len(ei) / (ms / 1e3)
        eot_base = {
            "kernel": "eot_pairs_kernel (per-pair n_i x n_j Gibbs kernel, SMEM or L2 slot)",
            "sample_pairs": int(len(ei)), "ms": ms, "pairs_per_s": rate,
            "whole_job_s_extrapolated": inp.n_pairs / rate,
            "asot_speedup": value / rate,
            "ground_cost": "normalised squared Euclidean on the original points (R#32)",
        }
        if da is not None:
            rel = np.abs(da - de) / np.maximum(de, 1e-3)
            eot_base.update({"asot_vs_eot_rmse": float(np.sqrt(np.mean((da - de) ** 2))),
                             "asot_vs_eot_rel_p50": float(np.median(rel)),
                             "asot_vs_eot_rel_p90": float(np.quantile(rel, 0.9)),
                             "eot_mean_distance": float(de.mean())})

    # ---- the explicit pair-list entry point on the same work (shuffled list of all i < j)
    pairs_api = None
    if args.pairs_api and rank == 0 and world == 1:
        _, Hq, _ = asot.map_to_anchors(pts, offs, w, anc, offsets_host=inp.offsets)
        iu, ju = np.triu_indices(inp.n_dist, k=1)
        perm = np.random.default_rng(5).permutation(iu.shape[0])
        qi, qj = t(iu[perm].astype(np.int32)), t(ju[perm].astype(np.int32))
        qst = asot.asot.new_status(dev)
        asot.pairwise_sinkhorn(Hq, cst, float(inp.eps), inp.iters, qi, qj, precision=prec, cost_max=cmax,
                               status=qst, workspace=ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dq = asot.pairwise_sinkhorn(Hq, cst, float(inp.eps), inp.iters, qi, qj, precision=prec,
                                    cost_max=cmax, status=qst, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        asot.check_status(qst)
        ms = e0.elapsed_time(e1)
        same = Dres[qi.long(), qj.long()]
        pairs_api = {"api": "asot_pairwise_sinkhorn (explicit shuffled list of all pairs)",
                     "ms": ms, "pairs_per_s": inp.n_pairs / (ms / 1e3),
                     "tflops": flops_per_pair * inp.n_pairs / (ms / 1e3) / 1e12,
                     "max_rel_diff_vs_tile_path": float(((dq - same).abs() / same.clamp_min(1e-3)).max())}

    # ---- NEXT-3: exact ASOT (eps -> 0 limit) on a pair sample, same GPU
    exact = None
    if args.exact and rank == 0 and world == 1:
        from asot_inputs import random_pairs
        _, Hx, _ = asot.map_to_anchors(pts, offs, w, anc, offsets_host=inp.offsets)
        # supports above 128 bins (K > 128 with dense histograms, e.g. c5) run the CTA-per-pair
        # solver at ~100 pairs/s: a smaller default sample there
        n_ex = args.exact_pairs if args.exact_pairs > 0 else (20000 if inp.n_anchors <= 128 else 1000)
        xi, xj = random_pairs(inp.n_dist, min(n_ex, inp.n_pairs), seed=78)
        xi_d, xj_d = t(xi.astype(np.int32)), t(xj.astype(np.int32))
        xst = asot.asot.new_status(dev)
        asot.exact_asot_pairs(Hx, cst, xi_d, xj_d, status=xst)      # warm-up
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d_ex = asot.exact_asot_pairs(Hx, cst, xi_d, xj_d, status=xst)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        dx = d_ex.cpu().numpy()
        ok = np.isfinite(dx)
        da = Dres.cpu().numpy()[xi, xj].astype(np.float64)
        rel = np.abs(da[ok] - dx[ok]) / np.maximum(dx[ok], 1e-3)
        exact = {"kernel": "exact_pairs_kernel (fp64 successive-shortest-path min-cost flow on the "
                           "histogram supports: warp per pair up to 128 bins, CTA per pair above)",
                 "sample_pairs": int(len(xi)), "solved": int(ok.sum()), "ms": ms,
                 "pairs_per_s": len(xi) / (ms / 1e3),
                 "easot_vs_exact_rmse": float(np.sqrt(np.mean((da[ok] - dx[ok]) ** 2))) if ok.any() else None,
                 "easot_vs_exact_rel_p50": float(np.median(rel)) if ok.any() else None,
                 "easot_vs_exact_rel_p90": float(np.quantile(rel, 0.9)) if ok.any() else None,
                 "support_limit": "none (K <= 1024)"}

    # ---- NEXT-3 bound checks: the paper's guarantee |W_AS - W_1| <= Prop. 1 / Prop. 2 bounds,
    # per pair at scale, all terms on the GPU (Euclidean C_s and C, R#7; one-hot P_o)
    bounds = None
    if args.bounds and rank == 0 and world == 1:
        from asot_inputs import random_pairs
        bi, bj = random_pairs(inp.n_dist, min(args.bounds_pairs, inp.n_pairs), seed=79)
        bi_d, bj_d = t(bi.astype(np.int32)), t(bj.astype(np.int32))
        bst = asot.asot.new_status(dev)
        asg, Hb, _ = asot.map_to_anchors(pts, offs, w, anc, offsets_host=inp.offsets)
        CsE = asot.mahalanobis_cost(anc, torch.eye(inp.dim, dtype=torch.float32, device=dev), normalize=False)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        w_as = asot.exact_asot_pairs(Hb, CsE, bi_d, bj_d, status=bst)
        ev[1].record()
        w1 = asot.exact_w1_points(pts, offs, w, bi_d, bj_d, status=bst)
        ev[2].record()
        l1, linf, p2 = asot.bound_terms(pts, offs, anc, asg, CsE, bi_d, bj_d, status=bst)
        ev[3].record()
        torch.cuda.synchronize()
        st_b = int(bst.item())
        w_as, w1 = w_as.cpu().numpy(), w1.cpu().numpy()
        l1, linf, p2 = l1.cpu().numpy(), linf.cpu().numpy(), p2.cpu().numpy()
        ok = np.isfinite(w1) & np.isfinite(w_as)
        gap = np.abs(w_as - w1)[ok]
        ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(3)]
        bounds = {
            "metric": "Euclidean C_s = ||w_u - w_v||_2 and C = ||x - y||_2 (R#7), one-hot P_o",
            "sample_pairs": int(len(bi)), "checked_pairs": int(ok.sum()),
            "skipped_w1_support_gt_64": int((~np.isfinite(w1)).sum()), "status_flags": st_b,
            "violations_prop1_l1": int((gap > l1[ok] + 1e-9).sum()),
            "violations_prop1_max": int((gap > linf[ok] + 1e-9).sum()),
            "violations_prop2": int((gap > p2[ok] + 1e-9).sum()),
            "gap_mean": float(gap.mean()) if ok.any() else None,
            "gap_over_prop1_max_median": float(np.median(gap / linf[ok])) if ok.any() else None,
            "gap_over_prop1_l1_median": float(np.median(gap / l1[ok])) if ok.any() else None,
            "gap_over_prop2_median": float(np.median(gap / p2[ok])) if ok.any() else None,
            "ms": {"exact_w_as": ms[0], "exact_w1_points": ms[1], "bound_terms": ms[2]},
            "pairs_per_s": {"exact_w_as": len(bi) / (ms[0] / 1e3), "exact_w1_points": len(bi) / (ms[1] / 1e3),
                            "bound_terms": len(bi) / (ms[2] / 1e3)},
        }

    # ---- e2e: host buffers through the public C-ABI host entry point (N = 1), or the
    # distributed public API with H2D / D2H inside the timed region (N > 1)
    e2e = None
    if world == 1 and (args.mapping != "onehot" or args.anchors != "seeded"):
        # soft mappings: the public Python API with pinned host inputs copied in and D copied out
        hp = torch.from_numpy(inp.points).pin_memory()
        hw_ = torch.from_numpy(inp.weights).pin_memory()
        ho = torch.from_numpy(inp.offsets).pin_memory()
        hD = torch.empty((inp.n_dist, inp.n_dist), dtype=torch.float32).pin_memory()
        e_ms = []
        for _ in range(args.e2e_steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            pts.copy_(hp, non_blocking=True); w.copy_(hw_, non_blocking=True)
            offs.copy_(ho, non_blocking=True)
            hD.copy_(step(), non_blocking=True)
            torch.cuda.synchronize()
            e_ms.append((time.perf_counter() - t0) * 1e3)
        e2e = {"value": P * len(e_ms) / (sum(e_ms) / 1e3), "unit": "pairs/s",
               "h2d_bytes_per_step": int(hp.numel() * 4 + hw_.numel() * 4 + ho.numel() * 8),
               "d2h_bytes_per_step": int(hD.numel() * 4),
               "api": ("paper_2310_16123_b200.kmeans_minibatch + sqeuclid_cost + distance_matrix"
                       if args.anchors == "kmeans" else
                       f"paper_2310_16123_b200.map_soft_{args.mapping} + distance_matrix(hist)")
                      + " (pinned host copies in, D out, wall clock)"}
    elif world == 1:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        hp, ho, hw, ha, hc = pin(inp.points), pin(inp.offsets), pin(inp.weights), pin(inp.anchors), pin(inp.cost)
        hD = torch.empty((inp.n_dist, inp.n_dist), dtype=torch.float32).pin_memory().numpy()
        wsh = asot.Workspace(dev)
        asot.distance_matrix_host(hp, ho, hw, ha, hc, float(inp.eps), inp.iters, precision=prec,
                                  out=hD, workspace=wsh)
        torch.cuda.synchronize()
        e_ms = []
        for _ in range(args.e2e_steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, st = asot.distance_matrix_host(hp, ho, hw, ha, hc, float(inp.eps), inp.iters,
                                              precision=prec, out=hD, workspace=wsh)
            e_ms.append((time.perf_counter() - t0) * 1e3)
            assert st == 0
        h2d = hp.nbytes + ho.nbytes + hw.nbytes + ha.nbytes + hc.nbytes
        d2h = hD.nbytes + 4
        e2e = {"value": P * len(e_ms) / (sum(e_ms) / 1e3), "unit": "pairs/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "api": "asot_distance_matrix_host (pinned host buffers, wall clock)"}
    else:
        hp = torch.from_numpy(inp.points).pin_memory()
        hw_ = torch.from_numpy(inp.weights).pin_memory()
        ha = torch.from_numpy(inp.anchors).pin_memory()
        hc = torch.from_numpy(inp.cost).pin_memory()
        ho = torch.from_numpy(inp.offsets).pin_memory()
        e_ms = []
        for _ in range(args.e2e_steps):
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            pts.copy_(hp, non_blocking=True); w.copy_(hw_, non_blocking=True)
            anc.copy_(ha, non_blocking=True); cst.copy_(hc, non_blocking=True)
            offs.copy_(ho, non_blocking=True)
            Dr = step()
            if rank == 0:
                Dr.cpu()
            torch.cuda.synchronize()
            dist.barrier()
            e_ms.append((time.perf_counter() - t0) * 1e3)
        tt = torch.tensor([sum(e_ms)], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        h2d = (hp.numel() * 4 + hw_.numel() * 4 + ha.numel() * 4 + hc.numel() * 4 + ho.numel() * 8) * world
        e2e = {"value": P * len(e_ms) / (float(tt[0]) / 1e3), "unit": "pairs/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(inp.n_dist ** 2 * 4),
               "api": "paper_2310_16123_b200.distributed (pinned host copies + D to host on rank 0)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.anchors == "seeded":
        v, sample = oracle_sample_rate(inp, args.cpu_budget, mapping=args.mapping, model=soft_model)
        cpu = {"value": v, "unit": "pairs/s", "cores": len(os.sched_getaffinity(0)),
               "kind": "oracle", "sample": sample}
        if eot_base is not None:
            # the paper's CPU comparison system, one pair at a time (Table 2 "eOT (CPU)"):
            # the fp64 eOT oracle on the GPU leg's seeded pairs until the budget, extrapolated
            from oracle import eot_oracle as EO
            done, t_eot = 0, 0.0
            while t_eot < args.cpu_budget / 2 and done < len(ei):
                s0 = time.perf_counter()
                EO.eot_pair_costs(inp.points, inp.offsets, inp.weights, float(inp.eps), inp.iters,
                                  ei[done:done + 16], ej[done:done + 16], scale)
                t_eot += time.perf_counter() - s0
                done += len(ei[done:done + 16])
            r_cpu = done / t_eot
            cpu["eot_one_by_one"] = {
                "pairs_per_s": r_cpu, "sample_pairs": done, "seconds": t_eot,
                "whole_job_s_extrapolated": inp.n_pairs / r_cpu,
                "gpu_eot_speedup": eot_base["pairs_per_s"] / r_cpu,
                "asot_speedup": value / r_cpu,
                "note": "fp64 eOT oracle (per-pair n_i x n_j cost + Sinkhorn, L iterations) on the "
                        "first pairs of the eOT leg's seeded sample"}

    if rank == 0:
        line = {
            "metric": baseline_metric(), "value": value, "unit": "pairs/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if kind == 11 else "tf32" if eff == asot.TF32 else ("f32 (3xtf32)" if kind in (3, 5) else
                                                      "f32 (bf16x3)" if kind == 10 else "f32"),
            "data": "synthetic",
            "config": workload_config(inp, args, world),
            "result_exchange": exchange_note[0],
            "roofline": roofline, "mapping": mapping, "kmeans": kmeans, "eot_baseline": eot_base,
            "exact_asot": exact, "pairs_api": pairs_api, "bounds": bounds,
            "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": gpu_launches,
            "gpu_launches_note": "launch-helper calls of libasot inside the timed region (a lower bound on "
                                 "kernels: each helper enqueues >= 1 of the library's kernels; the ncu "
                                 "launch list under profiles/ has every kernel of a step)",
            "clocks": clk,
            "wall_s_timed_region": wall,
            "env": asot_env(),
            "step_ms_min_median_max": [min(step_ms), statistics.median(step_ms), max(step_ms)],
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
