#!/usr/bin/env python
"""Benchmark of the EXACT hot path (arXiv 2503.19925) on B200.

One step = one EXACT iteration (Eq. extragrad-method):
2 loss+grad passes over A (K1) + 2 reduce/step/projection kernels (K2/K3),
replayed from a CUDA graph.  Metric (BASELINE.json): loss+grad A-stream GB/s
(whole job, all ranks) with iterations/s and the HBM-roofline fraction.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5|c2|c3|c4|c1f32]
  python bench.py --impl reference ...   # the fp64 oracle on host cores

The plain invocation runs C5 (n = 8e6, d = 4096, 131 GB: BASELINE.json
configs[4], the largest dense config, which fits one B200) at N = 1.

Multi-GPU: `--gpus N` without a torchrun environment re-launches this file
under torch.distributed.run with N ranks (127.0.0.1, one process per GPU,
NCCL_DEBUG=INFO into gpurun_out/); under torchrun the ranks read RANK /
LOCAL_RANK / WORLD_SIZE.  Rows are sharded across ranks with one cross-rank
sum of the d+1 vector per F evaluation.  c5/c4 scale strongly (the config's
rows are split), c2/c3 weakly (each rank holds the config's rows of a problem
N times larger).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
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
    "c5": "C5 large dense n=8e6 d=4096 W=32 fp32, 131 GB (BASELINE configs[4])",
}
STRONG = {"c5", "c4", "c1f32"}
DEFAULT_STEPS = {"c5": 20}
NOMINAL_HBM = 8000.0         # GB/s, BASELINE.json north_star "roughly 8 TB/s"
FALLBACK_HBM = 6650.0        # B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent
CPU_SLICE_ROWS = {"c5": 500_000}   # the C5 oracle leg streams a fixed 500k-row slice
METRIC = ("loss+grad A-stream GB/s (whole job; 1 step = 1 EXACT iteration = 2 loss+grad "
          "passes over A + 2 projections)")


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


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ------------------------------------------------------------------ clocks
class Clocks:
    """SM clock and throttle reasons sampled (NVML, every 5 ms) while the
    timed region runs (B200_PROFILING.md clocks line)."""

    NAMES = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
             "sw_power_cap": 0x4}

    def __init__(self, cuda_index):
        self.samples = []
        self.max_mhz = None
        self.h = None
        self._stop = threading.Event()
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            pr = torch.cuda.get_device_properties(cuda_index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            try:
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(cuda_index)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.h = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, rs))
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.h is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.h is not None:
            self._stop.set()
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return None
        reasons = sorted({n for _, rs in self.samples for n, bit in self.NAMES.items() if rs & bit})
        return {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "nvml, 5 ms"}


# ------------------------------------------------------------------ ranks
def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(args):
    """`--gpus N` outside torchrun: run this file under torch.distributed.run
    with N local ranks (one process per GPU) and forward its exit code."""
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_FILE", os.path.join(ROOT, "gpurun_out", "nccl_debug.%h.%p.log"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def dist_setup(backend="nccl"):
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            import torch
            # the library's own communicator reads these at ncclCommInitRank
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_FILE",
                                  os.path.join(ROOT, "gpurun_out", "nccl_debug.%h.%p.log"))
            os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
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


def kernel_label(w, poly):
    """The kernels of one loss+grad pass, by the layout poly_init chose."""
    if "A" in w:
        return "k_dense_loss_grad"
    lay = poly.describe().get("csr_layout", 1)
    return {3: "k_strip_forward+k_strip_link+k_tile_backward", 2: "k_dsell_forward+k_dsell_backward",
            1: "k_sell16_forward+k_sell16_backward"}.get(lay, "k_sell_forward+k_csc_backward")


def read_traffic(name):
    tpath = os.path.join(ROOT, "profiles", f"traffic_{name}.json")
    try:
        return json.load(open(tpath)).get("dram_bytes_per_launch")
    except Exception:
        return None


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist
    rank, world, local = dist_setup()
    torch.cuda.set_device(local)
    import paper_2503_19925_b200 as P
    from paper_2503_19925_b200 import dist as D
    from paper_2503_19925_b200 import workloads as PW

    cfg0 = G.CONFIGS[args.config]
    cfg, row0, n_local, scaling = D.shard(cfg0, rank, world, strong=cfg0.name in STRONG)
    w = PW.build(cfg, row0=row0, n_local=n_local)
    nccl_id = D.exchange_id(P.poly_nccl_unique_id, rank, world)
    p2p = args.p2p and world > 1
    nvls = args.nvls and world > 1
    flags = (P.POLY_FLAG_P2P if p2p else 0) | (P.POLY_FLAG_NVLS if nvls else 0)
    poly = PW.make_poly(w, rank=rank, world=world, nccl_id=nccl_id, flags=flags)
    if p2p:
        poly.p2p_setup()   # K9: cross-rank sum over NVLink peer memory instead of ncclAllReduce
    if nvls:
        poly.nvls_setup()  # K9-NVLS: cross-rank sum in the NVSwitch (multicast object)
    gamma = gamma_for(cfg)
    x = torch.zeros(cfg.d, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    def timed(profile):
        x.zero_()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        poly.solve(x, args.steps, gamma, profile=profile)
        e1.record(st)
        torch.cuda.synchronize()
        barrier()
        return e0.elapsed_time(e1)

    poly.solve(x, args.warmup, gamma)              # warm-up (graph capture happens here)
    clk = Clocks(local)
    with clk:
        ms_local = timed(False)
        # the same K iterations again, the same kernels and launch
        # configurations launched one by one on the same stream with CUDA
        # events around every kernel: the per-kernel times of the roofline
        # and the step time they are a share of come from this one run
        prof_ms = timed(True)
    kt = poly.kernel_times()
    ms = D.max_over_ranks(ms_local, world)
    ab = a_bytes(w)
    total_a = D.sum_over_ranks(float(ab), world)
    gbs = 2.0 * args.steps * total_a / (ms * 1e-3) / 1e9
    iters = args.steps / (ms * 1e-3)

    peak, peak_src = measured_peak()
    per_launch = ab + side_bytes(w)
    achieved = per_launch / (kt[0] * 1e-3) / 1e9 if kt[0] > 0 else None
    read_ceiling = None
    if "A" in w:   # K8: the same bytes through the same ring, no arithmetic
        read_ceiling = ab / (poly.stream_probe(5 if ab > 20e9 else 20) * 1e-3) / 1e9
    prof_step = prof_ms / args.steps
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": (achieved / peak) if achieved else None, "traffic": read_traffic(args.config),
            "peak_source": peak_src,
            "nominal_peak": NOMINAL_HBM, "frac_nominal": (achieved / NOMINAL_HBM) if achieved else None,
            "kernel": kernel_label(w, poly),
            "kernel_ms": kt[0], "finalize_ms": kt[1], "allreduce_ms": kt[2],
            "bytes_per_launch": per_launch,
            "timing": "CUDA events around every kernel of K iterations launched one by one on the solve's "
                      "stream (same kernels and launch configurations as the timed graph replays)",
            "instrumented_step_ms": prof_step,
            "step_share": (2 * kt[0]) / prof_step if prof_step > 0 else None,
            "read_ceiling_k8": read_ceiling,
            "frac_of_read_ceiling": (achieved / read_ceiling) if achieved and read_ceiling else None}
    desc = poly.describe()
    # part of A the kernels read with L2 evict-last: it stays in L2 from pass to pass, so the DRAM bytes of
    # a pass in the timed loop are below the algorithmic bytes by up to this much (`traffic` is ncu's
    # cold-cache figure); `achieved` stays algorithmic bytes / time
    roof["l2_keep_bytes"] = desc.get("l2_keep_bytes", 0)
    launches = launches_per_step(w, cfg, world) * args.steps  # (before e2e releases the device copy of A)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.config, w, seconds=args.cpu_seconds)
    poly.close()
    del poly   # drops the handle's references to A (C5: 131 GB that e2e needs back)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(P, D, w, cfg, gamma, args, rank, world)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": gbs, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Philox generators, BASELINE.json recipe)",
            "config": {"workload": WORKLOAD_DESC.get(args.config, args.config), "name": args.config,
                       "n_global": cfg.n, "n_local": n_local, "d": cfg.d, "W": cfg.W,
                       "I_bar": cfg.I_bar, "parallelism": "dp1 (single GPU, no collective)" if world == 1 else
                       f"dp{world} (row shards + " + ("K9 NVLink peer reduce)" if p2p else
                                                     "K9-NVLS switch reduce)" if nvls else "NCCL allreduce)"),
                       "precision": "fp32 A, fp32 FMA dot/axpy; fp64 link, residual, reductions, iterate",
                       "l2": "inputs larger than L2 (A >> 126 MB), no flush" if ab > 4 * 126e6 else
                             "A may be L2-resident (small shard)",
                       "gamma": gamma, "tile": desc},
            "iters_per_s": iters, "calls_per_s": 2 * iters,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if world > 1:
            line["nccl"] = {"comm_ranks": desc.get("comm_ranks"), "k9": desc.get("k9"),
                            "debug_log": os.environ.get("NCCL_DEBUG_FILE")}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(P, D, w, cfg, gamma, args, rank=0, world=1):
    """The same metric through the C ABI with HOST inputs: every step is
    poly_init(POLY_FLAG_HOST_INPUTS: A, y copied from pinned host memory into
    library-owned HBM; with N ranks each its row block and a fresh
    communicator) + poly_solve(T iterations from a host x, x returned to the
    host) + poly_free; the timed region covers all of it (max over ranks).
    The device copy of A made by the workload builder is released first (C5's
    131 GB would not fit twice)."""
    import psutil
    import torch
    ab = a_bytes(w)
    need = ab + side_bytes(w)
    # every rank of the node stages its block: the node must hold them all;
    # the decision is rank 0's, so that all ranks take the same path
    skip = need * world * 1.15 + 8e9 > psutil.virtual_memory().available
    if world > 1:
        skip = D.max_over_ranks(1.0 if skip else 0.0, world) > 0.5
    if skip:
        return {"value": None, "unit": "GB/s",
                "skipped": f"host memory: {need * world / 1e9:.0f} GB of inputs, "
                           f"{psutil.virtual_memory().available / 1e9:.0f} GB available"}
    cudart = torch.cuda.cudart()
    registered = []

    def pinned_copy(t):
        """Pinned host copy of device tensor t: plain host pages registered
        with cudaHostRegister (the caching pinned allocator would round a
        131 GB request up to 256 GB), filled by D2H copies in 1 GiB pieces."""
        h = torch.empty(t.shape, dtype=t.dtype)
        nb = h.numel() * h.element_size()
        if nb:
            rc = cudart.cudaHostRegister(h.data_ptr(), nb, 0)
            if int(rc) != 0:
                raise RuntimeError(f"cudaHostRegister({nb} bytes) failed: {rc}")
            registered.append(h)
        hf, tf = h.view(-1), t.reshape(-1)
        step = max(1, (1 << 30) // max(1, h.element_size()))
        for a in range(0, hf.numel(), step):
            hf[a:a + step].copy_(tf[a:a + step], non_blocking=True)
        torch.cuda.synchronize()
        return h

    t0 = time.perf_counter()
    y_h = pinned_copy(w["y"])
    if "A" in w:
        mat = dict(A=pinned_copy(w["A"]))
    else:   # CSR: the caller's arrays; poly_init builds the SELL copies on the device
        mat = dict(row_ptr=pinned_copy(w["row_ptr"]), col=pinned_copy(w["col"]), val=pinned_copy(w["val"]))
    extra = {}
    if w.get("s_row") is not None:
        extra = dict(s_row=pinned_copy(w["s_row"]), I_row=pinned_copy(w["I_row"]))
    prep_s = time.perf_counter() - t0
    for k in ("A", "row_ptr", "col", "val", "y", "counts", "lam", "s_row", "I_row", "mat"):
        w.pop(k, None)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    T = args.e2e_T or cfg.T
    st = torch.cuda.current_stream()
    vals = []
    steps = args.e2e_steps if ab < 20e9 else min(args.e2e_steps, 2)
    for rep in range(1 + steps):
        x_h = torch.zeros(cfg.d, dtype=torch.float64).pin_memory()
        nid = D.exchange_id(P.poly_nccl_unique_id, rank, world)   # a communicator per init
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        p = P.Poly(d=cfg.d, y=y_h, s=w["s"], mu=w["mu"], I_bar=cfg.I_bar, set=cfg.set,
                   R=w["R"], n_global=w["n_global"], row_offset=w["row0"], rank=rank, world=world,
                   nccl_id=nid, flags=P.POLY_FLAG_HOST_INPUTS, stream=st.cuda_stream, **mat, **extra)
        p.solve(x_h, T, gamma)
        e1.record(st)
        torch.cuda.synchronize()
        p.close()
        if rep > 0:                                  # rep 0 warms the allocator/graph path
            vals.append(D.max_over_ranks(e0.elapsed_time(e1), world))
    ms = statistics.median(vals)
    ab = D.sum_over_ranks(float(ab), world)
    h2d = D.sum_over_ranks(float(sum(v.numel() * v.element_size()
                                     for v in [y_h] + list(mat.values()) + list(extra.values()))), world)
    for h in registered:
        cudart.cudaHostUnregister(h.data_ptr())
    return {"value": 2.0 * T * ab / (ms * 1e-3) / 1e9, "unit": "GB/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 8 * cfg.d * world,
            "iterations_per_step": T, "ms_per_step": ms, "steps_timed": len(vals),
            "host_prep_s": prep_s,
            "note": "step = poly_init(pinned host A or CSR, y) + poly_solve(T, host x) + poly_free"}


# ------------------------------------------------------------------ the oracle on host cores
def oracle_slice(name, w=None, rows=None):
    """The oracle's copy of a bounded row sample of workload `name`: dense
    configs take the sample's generated rows from the device workload when one
    is given (the shared seeded generator's bytes, checked on sampled rows by
    oracle.workloads), else draw them with gen/rng; λ, counts and A.1 spectra
    are the oracle's own."""
    from oracle import workloads as OW
    cfg = G.CONFIGS[name]
    if cfg.kind == "csr":
        wo = OW.build(cfg)
        return wo, wo["val"].shape[0] * 8 + wo["row_ptr"].shape[0] * 8, "all rows (the CSR matrix)"
    m = rows or min(cfg.n, CPU_SLICE_ROWS.get(name, max(2048, int(2e8 // cfg.d))))
    idx = np.arange(m)
    A = K = None
    if w is not None and "A" in w and w.get("row0", 0) == 0 and w["n_local"] >= m:
        A = w["A"][:m, :cfg.d].cpu().numpy()
        if cfg.kind == "reparam":
            import torch
            from paper_2503_19925_b200 import synth
            from gen import rng
            Kt = torch.empty((m, 2 * cfg.d), dtype=torch.float32, device="cuda")
            synth.gaussian_matrix(Kt, 2 * cfg.d, 0, cfg.seed, rng.STREAM_A_KNOWN)
            K = Kt.cpu().numpy()
            del Kt
    wo = OW.build(cfg, rows=idx, A=A, A_known=K)
    return wo, m * cfg.d * 4, f"first {m} of {cfg.n} rows"


def cpu_baseline(name, w=None, seconds=15.0):
    """The oracle as it stands (fp64 C, OpenMP over fixed 4096-row chunks) on a
    bounded row sample of the same workload: GB/s of A (fp32 bytes) processed
    by loss+grad calls, with all host cores and with one core."""
    import oracle
    wo, nbytes, sample = oracle_slice(name, w)
    prob = wo["problem"]
    x = np.zeros(prob.d)

    def rate(threads, budget, min_calls):
        oracle.set_threads(threads)
        t0 = time.perf_counter()
        calls = 0
        while calls < min_calls or time.perf_counter() - t0 < budget:
            prob.F(x)
            calls += 1
        dt = time.perf_counter() - t0
        return calls * nbytes / dt / 1e9, calls, dt

    cores = len(os.sched_getaffinity(0))
    allc, n_all, t_all = rate(cores, seconds, 2)
    one, n_one, t_one = rate(1, seconds / 3, 1)
    oracle.set_threads(cores)
    return {"value": allc, "unit": "GB/s", "cores": cores, "kind": "oracle",
            "sample": f"{sample}; {n_all} loss+grad calls in {t_all:.1f} s",
            "calls_per_s": n_all / t_all, "cpu_model": cpu_model(), "nproc": os.cpu_count(),
            "one_core": {"value": one, "unit": "GB/s", "calls": n_one, "seconds": t_one}}


def run_reference(args):
    """--impl reference: the oracle's EXACT solve (Eq. extragrad-method) as it
    stands, on the host cores, over a bounded row sample of the workload; each
    step one EXACT iteration.  Under torchrun only rank 0 runs."""
    rank = env_int("RANK", 0)
    if rank != 0:
        return
    import oracle
    cfg = G.CONFIGS[args.config]
    w = None
    try:
        import torch
        if torch.cuda.is_available() and cfg.kind == "dense":
            from paper_2503_19925_b200 import synth
            from gen import rng
            m = min(cfg.n, CPU_SLICE_ROWS.get(args.config, max(2048, int(2e8 // cfg.d))))
            A = torch.empty((m, cfg.d), dtype=torch.float32, device="cuda")
            synth.gaussian_matrix(A, cfg.d, 0, cfg.seed, rng.STREAM_A)   # the shared seeded generator
            w = {"A": A, "row0": 0, "n_local": m}
    except Exception:
        w = None
    wo, nbytes, sample = oracle_slice(args.config, w)
    prob = wo["problem"]
    oracle.set_threads(len(os.sched_getaffinity(0)))   # torchrun exports OMP_NUM_THREADS=1
    gamma = gamma_for(cfg)
    x = np.zeros(cfg.d)
    x, _, _ = prob.solve(args.warmup, gamma, x1=x)
    t0 = time.perf_counter()
    x, _, _ = prob.solve(args.steps, gamma, x1=x)
    dt = time.perf_counter() - t0
    v = 2.0 * args.steps * nbytes / dt / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s",
            "n_gpus": env_int("WORLD_SIZE", 1), "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "strong" if args.config in STRONG else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD_DESC.get(args.config, args.config), "name": args.config,
                       "sample": sample},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": oracle.max_threads(),
                             "kind": "oracle", "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_mock(args):
    """--mock (CPU tests): the rank plumbing of run_ours with the library
    calls replaced by a gloo barrier — proves that `--gpus N` starts N ranks
    and that rank 0 alone reports."""
    import torch.distributed as dist
    rank, world, _ = dist_setup(backend="gloo")
    from paper_2503_19925_b200 import dist as D
    cfg0 = G.CONFIGS[args.config]
    cfg, row0, n_local, scaling = D.shard(cfg0, rank, world, strong=cfg0.name in STRONG)
    if world > 1:
        dist.barrier()
    total = D.sum_over_ranks(float(n_local), world, device="cpu")
    if rank == 0:
        print(json.dumps({"mock": True, "n_gpus": world, "rows_total": total, "scaling": scaling,
                          "nccl_debug": os.environ.get("NCCL_DEBUG")}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c5", choices=sorted(WORKLOAD_DESC))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--p2p", action="store_true",
                    help="N>1: sum over ranks with the K9 peer-reduce kernel instead of ncclAllReduce")
    ap.add_argument("--nvls", action="store_true",
                    help="N>1: sum over ranks in the NVSwitch (K9-NVLS multicast kernel) instead of ncclAllReduce")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--e2e-T", type=int, default=0)
    ap.add_argument("--mock", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.steps is None:
        args.steps = DEFAULT_STEPS.get(args.config, 200)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.mock:
        run_mock(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
