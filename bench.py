#!/usr/bin/env python
"""Benchmark of the EXACT hot path (arXiv 2503.19925) on B200.

One step = one EXACT iteration (Eq. extragrad-method):
2 loss+grad passes over A (K1) + 2 reduce/step/projection kernels (K2/K3),
replayed from a CUDA graph.  Metric (BASELINE.json): loss+grad A-stream GB/s
(whole job, all ranks) with iterations/s and the HBM-roofline fraction.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c4|c5|c1f32]
  python bench.py --impl reference ...   # the fp64 oracle on host cores

Multi-GPU (torchrun, one process per GPU, NCCL): rows are sharded across
ranks with one ncclAllReduce of the d-vector per F evaluation.  c2/c3 scale
weakly (each rank holds the config's full row count of a problem N times
larger); c5 scales strongly (its 8e6 rows are split).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from gen import configs as G  # noqa: E402

WORKLOAD_DESC = {
    "c1f32": "C1 tiny dense n=2000 d=100 W=10 fp32 (BASELINE configs[0])",
    "c2": "C2 medium dense n=200000 d=1024 W=20 fp32 Gaussian (BASELINE configs[1])",
    "c3": "C3 three-material reduced model n=1e6 d=512 W=16 per-row spectra (BASELINE configs[2])",
    "c4": "C4 CT-like CSR 256x256 image, 360x367 rays, W=16, fp32 y with noise (BASELINE configs[3])",
    "c5": "C5 large dense n=8e6 d=4096 W=32 fp32 (BASELINE configs[4])",
}
STRONG = {"c5", "c4", "c1f32"}
FALLBACK_HBM = 6650.0


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{index}.csv")

    def __enter__(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "20"], stdout=self.f,
                stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines()]
        except Exception:
            return None
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [v.strip() for v in r]
            if len(r) < 8:
                continue
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except ValueError:
                continue
            for nm, v in zip(names, r[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup(args):
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def gamma_for(cfg):
    """Theorem 2 step 1/(4 Ī λmax(Σ) Σ s_j μ_j) (reading R5) with
    λmax from the Marchenko–Pastur edge (1 + sqrt(d/n))² for Gaussian A; the
    throughput does not depend on γ."""
    s, mu = cfg.spectrum
    if cfg.kind == "csr":
        lam = 2e-5
    else:
        lam = (1.0 + math.sqrt(cfg.d / cfg.n)) ** 2
    return 1.0 / (4.0 * cfg.I_bar * lam * float(np.dot(s, mu)))


def launches_per_step(w, cfg, world):
    """Our kernels per EXACT iteration (2 F evaluations): the pass (K1, or
    K4f + K4b), the reduce/step kernel, + k_fin_apply when d > 8192, and with
    world > 1 a REDUCE kernel per evaluation (the NCCL allreduce kernel is the
    library's, not counted)."""
    per_eval = (1 if "A" in w else 2) + 1 + (1 if cfg.d > 8192 else 0) + (1 if world > 1 else 0)
    return 2 * per_eval


def a_bytes(w):
    if "A" in w:
        n, d = w["n_local"], w["cfg"].d
        return n * d * w["A"].element_size()
    return w["val"].numel() * (w["val"].element_size() + 4) + w["row_ptr"].numel() * 8


def side_bytes(w):
    b = w["y"].numel() * w["y"].element_size()
    if w.get("s_row") is not None:
        b += w["s_row"].numel() * 4 + w["I_row"].numel() * 4
    return b


def run_ours(args):
    import torch
    import torch.distributed as dist
    rank, world, local = dist_setup(args)
    torch.cuda.set_device(local)
    import paper_2503_19925_b200 as P
    from paper_2503_19925_b200 import workloads as PW

    from paper_2503_19925_b200 import dist as D

    cfg0 = G.CONFIGS[args.config]
    cfg, row0, n_local, scaling = D.shard(cfg0, rank, world, strong=cfg0.name in STRONG)
    w = PW.build(cfg, row0=row0, n_local=n_local)
    nccl_id = D.exchange_id(P.poly_nccl_unique_id, rank, world)
    p2p = args.p2p and world > 1
    poly = PW.make_poly(w, rank=rank, world=world, nccl_id=nccl_id, flags=P.POLY_FLAG_P2P if p2p else 0)
    if p2p:
        poly.p2p_setup()   # K9: cross-rank sum over NVLink peer memory instead of ncclAllReduce
    gamma = gamma_for(cfg)
    x = torch.zeros(cfg.d, dtype=torch.float64, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()

    poly.solve(x, args.warmup, gamma)              # warm-up (graph capture happens here)
    x.zero_()
    barrier()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        e0.record(st)
        poly.solve(x, args.steps, gamma)
        e1.record(st)
        torch.cuda.synchronize()
    barrier()
    ms = D.max_over_ranks(e0.elapsed_time(e1), world)
    ab = a_bytes(w)
    total_a = D.sum_over_ranks(float(ab), world)
    gbs = 2.0 * args.steps * total_a / (ms * 1e-3) / 1e9
    iters = args.steps / (ms * 1e-3)

    # roofline of the dominant kernel (K1): event-timed profile pass, same K
    x.zero_()
    poly.solve(x, args.steps, gamma, profile=True)
    kt = poly.kernel_times()
    peak, peak_src = measured_peak()
    per_launch = ab + side_bytes(w)
    achieved = per_launch / (kt[0] * 1e-3) / 1e9 if kt[0] > 0 else None
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    read_ceiling = None
    if "A" in w:   # K8: the same bytes through the same ring, no arithmetic
        read_ceiling = ab / (poly.stream_probe(20) * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "kernel": "k_dense_loss_grad" if "A" in w else "k_csr_loss_grad",
            "kernel_ms": kt[0], "finalize_ms": kt[1], "allreduce_ms": kt[2],
            "bytes_per_launch": per_launch, "peak_source": peak_src,
            "read_ceiling_k8": read_ceiling,
            "frac_of_read_ceiling": (achieved / read_ceiling) if achieved and read_ceiling else None,
            "step_share": (2 * kt[0]) / (ms / args.steps) if ms > 0 else None}

    e2e = None
    if not args.no_e2e and world == 1:
        e2e = run_e2e(P, PW, w, cfg, gamma, args)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.config, seconds=args.cpu_seconds)

    if rank == 0:
        desc = poly.describe()
        clocks = clk.summary()
        line = {
            "metric": "loss+grad A-stream GB/s (whole job; 1 step = 1 EXACT iteration = 2 loss+grad "
                      "passes over A + 2 projections)",
            "value": gbs, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Philox generators, BASELINE.json recipe)",
            "config": {"workload": WORKLOAD_DESC.get(args.config, args.config), "name": args.config,
                       "n_global": cfg.n, "n_local": n_local, "d": cfg.d, "W": cfg.W,
                       "I_bar": cfg.I_bar, "parallelism": "dp1 (single GPU, no collective)" if world == 1 else
                       f"dp{world} (row shards + " + ("K9 NVLink peer reduce)" if p2p else "NCCL allreduce)"),
                       "precision": "fp32 A, fp32 FMA dot/axpy; fp64 link, residual, reductions, iterate",
                       "l2": "inputs larger than L2 (A >> 126 MB), no flush" if ab > 4 * 126e6 else
                             "A may be L2-resident (small shard)",
                       "gamma": gamma, "tile": desc},
            "iters_per_s": iters, "calls_per_s": 2 * iters,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step(w, cfg, world) * args.steps,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    poly.close()
    if world > 1:
        dist.destroy_process_group()


def run_e2e(P, PW, w, cfg, gamma, args):
    """Same metric through the C ABI with HOST inputs: poly_init copies A, y
    (pinned) to the device, poly_solve runs T iterations from a host x and
    returns x to the host; the timed region covers all of it."""
    import torch
    try:
        import psutil
        host_ok = a_bytes(w) * 1.5 < psutil.virtual_memory().available and a_bytes(w) < 48e9
    except Exception:
        host_ok = a_bytes(w) < 32e9
    if not host_ok:   # C5: a 131 GB pinned host copy of A does not fit the host
        return {"value": None, "unit": "GB/s", "skipped": "A does not fit in host memory"}
    y_h = w["y"].cpu().pin_memory()
    if "A" in w:
        A_h = w["A"].cpu().pin_memory()
        mat = dict(A=A_h)
    else:   # CSR: the caller's arrays; poly_init builds the SELL copies on the device
        mat = dict(row_ptr=w["row_ptr"].cpu().pin_memory(), col=w["col"].cpu().pin_memory(),
                   val=w["val"].cpu().pin_memory())
    extra = {}
    if w.get("s_row") is not None:
        extra = dict(s_row=w["s_row"].cpu().pin_memory(), I_row=w["I_row"].cpu().pin_memory())
    T = args.e2e_T or cfg.T
    vals = []
    st = torch.cuda.current_stream()
    for rep in range(1 + args.e2e_steps):
        x_h = torch.zeros(cfg.d, dtype=torch.float64).pin_memory()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        p = P.Poly(d=cfg.d, y=y_h, s=w["s"], mu=w["mu"], I_bar=cfg.I_bar, set=cfg.set,
                   R=w["R"], n_global=w["n_global"], flags=P.POLY_FLAG_HOST_INPUTS,
                   stream=st.cuda_stream, **mat, **extra)
        p.solve(x_h, T, gamma)
        e1.record(st)
        torch.cuda.synchronize()
        p.close()
        if rep > 0:                                  # rep 0 warms the allocator/graph path
            vals.append(e0.elapsed_time(e1))
    ms = statistics.median(vals)
    ab = a_bytes(w)
    h2d = y_h.numel() * y_h.element_size() + \
        sum(v.numel() * v.element_size() for v in list(mat.values()) + list(extra.values()))
    return {"value": 2.0 * T * ab / (ms * 1e-3) / 1e9, "unit": "GB/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 8 * cfg.d,
            "iterations_per_step": T, "ms_per_step": ms,
            "note": "step = poly_init(host A or CSR, y) + poly_solve(T, host x) + free"}


def cpu_baseline(name, seconds=15.0, max_rows=None):
    """The oracle as it stands (fp64 C, OpenMP over fixed chunks) on a bounded
    row sample of the same workload; GB/s of A (fp32 bytes) processed per
    second by loss+grad calls."""
    import oracle
    from oracle import workloads as OW
    cfg = G.CONFIGS[name]
    if cfg.kind == "csr":
        w = OW.build(cfg)
        nbytes = w["val"].shape[0] * 8 + (w["row_ptr"].shape[0]) * 8
        sample = "all rows"
    else:
        m = max_rows or min(cfg.n, max(2048, int(2e7 // cfg.d)))
        rows = np.arange(m)
        w = OW.build(cfg, rows=rows)
        nbytes = m * cfg.d * 4
        sample = f"first {m} of {cfg.n} rows"
    prob = w["problem"]
    x = np.zeros(cfg.d)
    t0 = time.perf_counter()
    calls = 0
    while True:
        prob.F(x)
        calls += 1
        if time.perf_counter() - t0 >= seconds:
            break
    dt = time.perf_counter() - t0
    return {"value": calls * nbytes / dt / 1e9, "unit": "GB/s", "cores": oracle.max_threads(),
            "kind": "oracle", "sample": f"{sample}; {calls} loss+grad calls in {dt:.1f} s",
            "calls_per_s": calls / dt}


def run_reference(args):
    rank = env_int("RANK", 0)
    if rank != 0:
        return
    import oracle
    from oracle import workloads as OW
    cfg = G.CONFIGS[args.config]
    m = min(cfg.n, max(2048, int(2e7 // cfg.d))) if cfg.kind != "csr" else cfg.n
    w = OW.build(cfg, rows=np.arange(m) if cfg.kind != "csr" else None)
    prob = w["problem"]
    nbytes = (m * cfg.d * 4) if cfg.kind != "csr" else w["val"].shape[0] * 8 + w["row_ptr"].shape[0] * 8
    gamma = gamma_for(cfg)
    x = np.zeros(cfg.d)
    x, _, _ = prob.solve(args.warmup, gamma, x1=x)
    t0 = time.perf_counter()
    x, _, _ = prob.solve(args.steps, gamma, x1=x)
    dt = time.perf_counter() - t0
    v = 2.0 * args.steps * nbytes / dt / 1e9
    line = {"impl": "reference", "metric": "loss+grad A-stream GB/s (whole job; 1 step = 1 EXACT "
            "iteration = 2 loss+grad passes over A + 2 projections)", "value": v, "unit": "GB/s",
            "n_gpus": env_int("WORLD_SIZE", 1), "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD_DESC.get(args.config, args.config), "name": args.config,
                       "sample_rows": m},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": oracle.max_threads(),
                             "kind": "oracle", "sample": f"first {m} rows of {args.config}"},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=600)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(WORKLOAD_DESC))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--p2p", action="store_true",
                    help="N>1: sum over ranks with the K9 peer-reduce kernel instead of ncclAllReduce")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--e2e-T", type=int, default=0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
