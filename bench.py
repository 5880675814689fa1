#!/usr/bin/env python3
"""Benchmark of the B200 KIFMM elastic matvec (the hot path of arXiv:1612.04082, Sec. 2.2).

One step = one fmm_matvec (single + double layer, kernel UP) over the 1M-point beam
surface (BASELINE.json configs[2] recipe scaled to N = 1,000,000; p = 6; 64 points per
leaf) with the tree already built -- "Single FMM pass (without tree construction)",
PAPER.md line 251 -- i.e. the operator applied at every GMRES iteration.

Output: one JSON line (rank 0).  Extra objects: `phases` (native per-phase device
time and roofline fraction), `p2p` (direct all-pairs double-layer kernel on configs[1],
Ginteractions/s and fraction of FP32 peak), `roofline` (dominant phase), `cpu_baseline`
(the fp64 oracle direct sum timed on the host cores on a bounded target sample; the
same sample gives the GPU result's relative L2 error `rel_l2`), `e2e` (host buffers,
copies inside the timed region), `clocks`.

`--impl reference` times the oracle (fp64 C direct sum, the plain definition of
Eq. fmm_summation) on the host cores on bounded target samples of the same workload.
Multi-GPU (torchrun): replicas only -- every rank runs the same independent matvec
(DESIGN.md Sec. 8(e)); the timed region is barrier-bracketed and the max over ranks
is reported.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
METRIC = "elastic P2P Ginteractions/s (% FP32 peak); FMM matvec ms at N=1M, rel-L2 err"
WORKLOAD = "beam4x1x1_surface_N1M_graded_UP_kifmm_p6_leaf64"


def peaks():
    try:
        d = json.load(open(PEAKS_FILE))
        src = "measured"
    except Exception:
        d = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}
        src = "fallback"
    clk = d.get("sm_max_mhz", 1965.0) * 1e6
    # FP32: 148 SMs x 128 FFMA lanes x 2 flops x max SM clock; FP64: 64 lanes (B200 guide);
    # TF32 tensor: the measured bf16 GEMM peak x the guide's nominal dense ratio 1.1 / 2.25
    return dict(src=src, hbm_gbs=d["hbm_gbs"], fp32_tflops=148 * 128 * 2 * clk / 1e12,
                fp64_tflops=148 * 64 * 2 * clk / 1e12, tf32_tflops=d["bf16_tflops"] * 1.1 / 2.25,
                bf16_tflops=d["bf16_tflops"])


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: NVML polled every 5 ms
    from a thread (the timed matvec loop lasts ~0.1 s, too short for nvidia-smi's 50 ms
    sampling to see more than one or two samples), nvidia-smi -lms 50 if NVML is missing."""

    _BITS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
             0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []
        self.nv = None
        self.samples = []

    def _poll(self):
        import pynvml
        while not self.stop:
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, rs))
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(int(self.index))
            self.mx = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.stop = False
            self.nv = threading.Thread(target=self._poll, daemon=True)
            self.nv.start()
            return self
        except Exception:
            self.nv = None
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.nv is not None:
            self.stop = True
            self.nv.join(timeout=2)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.nv is not None:
            sm = [x for x, _ in self.samples]
            reasons = sorted({n for _, r in self.samples for b, n in self._BITS.items() if r & b})
            return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": float(self.mx),
                    "reasons": reasons, "samples": len(sm), "source": "nvml 5 ms"}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi 50 ms"}


def max_over_ranks(value, dist=None):
    """max of a per-rank timing over all ranks (device tensor under NCCL, host under gloo)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def workload(n):
    from workloads import geometry as geo
    return geo.config2(n=n)


_F64 = {}


def oracle_sample(d, sample_idx):
    """fp64 oracle (C direct sum) at the sampled targets; returns (values, seconds, threads).
    The fp64 copies of the inputs are made once (not timed: input marshalling)."""
    from oracle import cdirect
    from oracle import kernels as KN
    if id(d) not in _F64:
        _F64[id(d)] = {k: np.ascontiguousarray(d[k], np.float64) for k in ("src", "trg", "w", "f", "g", "nrm")}
    e = _F64[id(d)]
    trg = np.ascontiguousarray(e["trg"][sample_idx])
    t0 = time.perf_counter()
    ref = cdirect.direct_sum(KN.KERNEL_UP, trg, e["src"], d["K"], d["G"], w=e["w"], f=e["f"], g=e["g"], nrm=e["nrm"])
    return ref, time.perf_counter() - t0, int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))


def run_reference(args):
    """--impl reference: the oracle timed on the host cores, bounded samples per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    d = workload(args.n)
    n = d["trg"].shape[0]
    rng = np.random.default_rng(123)
    per_step = args.ref_sample
    times = []
    for k in range(args.warmup + args.steps):
        idx = np.sort(rng.choice(n, per_step, replace=False))
        _, sec, cores = oracle_sample(d, idx)
        if k >= args.warmup:
            times.append(sec * n / per_step)
    ms = 1e3 * float(np.mean(times))
    line = {"impl": "reference", "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n_points": n, "kernel": "UP", "method": "oracle direct sum (fp64 C)"},
            "cpu_baseline": {"value": ms, "unit": "ms", "cores": cores, "kind": "oracle",
                             "sample": f"{per_step} random targets x all {n} sources per step, "
                                       f"extrapolated to all {n} targets"},
            "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def p2p_bench(eb, torch, pk, reps=20):
    """configs[1]: direct double-layer traction kernel on the 24,576-triangle cube, all pairs."""
    from workloads import geometry as geo
    d = geo.config1()
    t = {k: torch.from_numpy(v).cuda() for k, v in d.items() if isinstance(v, np.ndarray)}
    n = d["src"].shape[0]
    out = torch.empty((n, 3), device="cuda")
    for _ in range(3):
        eb.bem_kernel_direct(eb.KERNEL_P, t["src"], t["src"], nrm=t["nrm"], w=t["w"], g=t["g"], K=d["K"], G=d["G"],
                             out=out)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        eb.bem_kernel_direct(eb.KERNEL_P, t["src"], t["src"], nrm=t["nrm"], w=t["w"], g=t["g"], K=d["K"], G=d["G"],
                             out=out)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    inter = float(n) * (n - 1)
    flops = inter * 45.0          # P kernel: FFMA=2, FMUL/FADD=1 in the compiled pair loop (tools/count_flops.sh)
    tf = flops / (ms * 1e-3) / 1e12
    res = {"config": "configs[1] cube 24576 triangles, kernel P, all pairs", "ms": ms,
           "ginteractions_per_s": inter / (ms * 1e-3) / 1e9, "tflops": tf,
           "frac_fp32_peak": tf / pk["fp32_tflops"], "flops_per_interaction": 45}
    # the same kernel on configs[2]'s 200k beam points (all 4e10 pairs): the sustained rate
    # without configs[1]'s small-problem tail and block reduction
    d2 = geo.config2(n=200_000, seed=0)
    t2 = {k: torch.from_numpy(v).cuda() for k, v in d2.items() if isinstance(v, np.ndarray)}
    n2 = d2["src"].shape[0]
    out2 = torch.empty((n2, 3), device="cuda")
    eb.bem_kernel_direct(eb.KERNEL_P, t2["src"], t2["src"], nrm=t2["nrm"], w=t2["w"], g=t2["g"], K=d2["K"],
                         G=d2["G"], out=out2)
    torch.cuda.synchronize()
    s.record()
    for _ in range(3):
        eb.bem_kernel_direct(eb.KERNEL_P, t2["src"], t2["src"], nrm=t2["nrm"], w=t2["w"], g=t2["g"], K=d2["K"],
                             G=d2["G"], out=out2)
    e.record()
    torch.cuda.synchronize()
    ms2 = s.elapsed_time(e) / 3
    tf2 = float(n2) * (n2 - 1) * 45.0 / (ms2 * 1e-3) / 1e12
    res["large"] = {"config": f"configs[2] beam {n2} points, kernel P, all pairs", "ms": ms2,
                    "ginteractions_per_s": float(n2) * (n2 - 1) / (ms2 * 1e-3) / 1e9, "tflops": tf2,
                    "frac_fp32_peak": tf2 / pk["fp32_tflops"]}
    return res


def gmres_workload(args, eb, torch, emit=True, precond=None):
    """configs[4]: mixed-BVP BEM GMRES solve on the metamaterial cell (64 voids, ~1.93M
    triangles), restart 50, tol 1e-6, p = 8.  Reports iterations, solve time (device
    events), operator set-up time, the residual history (true |b - A x| / |b| at every
    restart) and the global equilibrium of the solved tractions (sum of traction x area over
    the closed surface; exact solution: 0).  PAPER.md l. 250-251 reports the surface solve."""
    from workloads import geometry as geo
    precond = args.precond if precond is None else precond
    d = geo.metamaterial_cell(nc=args.cell_nc, level=args.cell_level, nvoids=args.cell_voids)
    verts = torch.from_numpy(d["verts"]).cuda()
    bc = torch.from_numpy(d["bc_type"]).cuda()
    val = torch.from_numpy(d["bc_val"]).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op = eb.bem_create(verts, nq=args.nq, max_pts=args.gmres_max_pts, p=args.gmres_p, K=d["K"], G=d["G"])
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    x = torch.zeros((d["verts"].shape[0], 3), device="cuda")
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = eb.ebem_launch_count()
    with ClockSampler(args.smi_index) as clk:
        a.record()
        x, it, res = eb.bem_gmres_solve(op, bc, val, x, restart=50, max_iter=args.max_iter, tol=1e-6,
                                        precond=precond, check=False)
        b.record()
        torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    est, true = eb.bem_gmres_history(op)
    V = d["verts"].astype(np.float64)
    area = 0.5 * np.linalg.norm(np.cross(V[:, 1] - V[:, 0], V[:, 2] - V[:, 0]), axis=1)
    t = np.where(d["bc_type"][:, None] == 0, x.cpu().numpy(), d["bc_val"])
    force = (t * area[:, None]).sum(0)
    del op
    torch.cuda.empty_cache()
    line = {"metric": "BEM GMRES solve time (configs[4])", "value": ms / 1e3, "unit": "s", "n_gpus": 1,
            "steps": 1, "warmup": 0, "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 FMM, f64 Krylov", "data": "synthetic",
            "config": {"workload": f"metamaterial cell, {d['verts'].shape[0]} triangles, {args.cell_voids} voids",
                       "nq": args.nq, "p": args.gmres_p, "max_pts": args.gmres_max_pts, "restart": 50, "tol": 1e-6,
                       "precond": ["none (paper)", "block-Jacobi 3x3 (right)", "leaf-block Jacobi (right)"][precond]},
            "converged": bool(res <= 1e-6), "iterations": it, "rel_residual": res,
            "ms_per_iteration": ms / max(it, 1), "setup_s": setup,
            "true_residual_at_restarts": [float(v) for v in true],
            "gpu_launches": int(eb.ebem_launch_count() - launches0),
            "equilibrium_residual": float(np.linalg.norm(force)), "applied_load": 1.0, "clocks": clk.summary()}
    if emit:
        print(json.dumps(line), flush=True)
    return line


def stress_workload(args, eb, torch, emit=True):
    """configs[3]: stress (D + S) of 500k beam-surface sources with smooth densities at 1M
    interior grid targets, p = 8: the topological-derivative evaluation (
    l. 250-251 report the volume evaluation).  Device time per evaluation (L2-flushed steps),
    tree build time, rel-L2 and the worst sampled target on 1000 targets vs the fp64 oracle."""
    from oracle import cdirect
    from oracle import kernels as KN
    from workloads import geometry as geo
    d = geo.config3()
    t = {k: torch.from_numpy(np.ascontiguousarray(v, np.float32)).cuda() for k, v in d.items()
         if isinstance(v, np.ndarray)}
    eb.fmm_build_tree(t["src"], t["nrm"], t["w"], trg=t["trg"], max_pts=args.stress_max_pts, p=args.stress_p,
                      K=d["K"], G=d["G"])          # first build: translation operators of this order
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tree = eb.fmm_build_tree(t["src"], t["nrm"], t["w"], trg=t["trg"], max_pts=args.stress_max_pts,
                             p=args.stress_p, K=d["K"], G=d["G"])
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    nt = d["trg"].shape[0]
    out = torch.empty((nt, 6), device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(max(args.warmup, 3)):
        eb.fmm_eval_stress(tree, eb.KERNEL_DS, t["f"], t["g"], out=out)
    torch.cuda.synchronize()
    steps = max(args.steps, 5)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    launches0 = eb.ebem_launch_count()
    with ClockSampler(args.smi_index) as clk:
        for k in range(steps):
            flush.fill_(float(k))
            ev[k][0].record()
            eb.fmm_eval_stress(tree, eb.KERNEL_DS, t["f"], t["g"], out=out)
            ev[k][1].record()
        torch.cuda.synchronize()
    launches = (eb.ebem_launch_count() - launches0) // steps
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    idx = np.sort(np.random.default_rng(11).choice(nt, 1000, replace=False))
    ref = cdirect.direct_sum(KN.KERNEL_DS, d["trg"][idx], d["src"], d["K"], d["G"], w=d["w"], f=d["f"], g=d["g"],
                             nrm=d["nrm"])
    got = out.cpu().numpy()[idx].astype(np.float64)
    rel = KN.rel_l2(got, ref)
    worst = float(np.linalg.norm(got - ref, axis=1).max() / np.linalg.norm(ref, axis=1).max())
    del tree
    torch.cuda.empty_cache()
    line = {"metric": "FMM stress evaluation ms (configs[3])", "value": ms, "unit": "ms", "n_gpus": 1,
            "steps": steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 (fp64 plan / equivalent densities)",
            "data": "synthetic",
            "config": {"workload": f"beam surface {d['src'].shape[0]} sources, {nt} interior grid targets, "
                                   "kernel D+S (6-component stress)", "p": args.stress_p,
                       "max_pts": args.stress_max_pts, "l2": "flushed between steps (256 MB write)"},
            "rel_l2": rel, "worst_target": worst, "oracle_sample": "1000 seeded targets, fp64 C direct sum",
            "tree_build_s": build_s, "targets_per_s": nt / (ms * 1e-3), "gpu_launches": launches,
            "clocks": clk.summary()}
    if emit:
        print(json.dumps(line), flush=True)
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--p", type=int, default=None, help="multipole order (default: 6 matvec, 8 gmres)")
    ap.add_argument("--max-pts", type=int, default=None,
                    help="leaf capacity (default: 64 for the matvec (configs[2]), 1536 for gmres)")
    ap.add_argument("--ref-sample", type=int, default=512)
    ap.add_argument("--cpu-sample", type=int, default=3072)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-p2p", action="store_true")
    ap.add_argument("--no-p10", action="store_true", help="skip the p = 10 line (configs[2]'s second order)")
    ap.add_argument("--workload", default="matvec", choices=["matvec", "gmres", "stress"])
    ap.add_argument("--nq", type=int, default=16)
    ap.add_argument("--cell-nc", type=int, default=160)
    ap.add_argument("--cell-level", type=int, default=5)
    ap.add_argument("--cell-voids", type=int, default=64)
    ap.add_argument("--max-iter", type=int, default=1000)
    ap.add_argument("--precond", type=int, default=2,
                    help="GMRES: 2 leaf-block Jacobi right preconditioner (default), 1 3x3 block-Jacobi, "
                         "0 the paper's plain GMRES")
    ap.add_argument("--no-stress", action="store_true", help="skip the configs[3] key of the matvec line")
    ap.add_argument("--no-gmres", action="store_true", help="skip the configs[4] key of the matvec line")
    ap.add_argument("--no-gmres-paper", action="store_true",
                    help="skip the configs[4] solve by the paper's unpreconditioned GMRES(50) (~2 min)")
    args = ap.parse_args()
    # leaf sizes / orders: configs[2] fixes 64 points per leaf for the matvec; configs[3] and
    # configs[4] state p = 8 and no leaf size: the fastest measured
    args.stress_max_pts = args.max_pts if (args.workload == "stress" and args.max_pts) else 256
    args.gmres_max_pts = args.max_pts if (args.workload == "gmres" and args.max_pts) else 1536
    args.stress_p = args.p if (args.workload == "stress" and args.p) else 8
    args.gmres_p = args.p if (args.workload == "gmres" and args.p) else 8
    if args.max_pts is None:
        args.max_pts = 64
    if args.p is None:
        args.p = 6
    if args.impl == "reference":
        return run_reference(args)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    ids = vis.split(",") if vis else [str(i) for i in range(64)]
    smi_index = ids[local]                       # nvidia-smi uses physical indices
    args.smi_index = smi_index
    if world > 1:
        # one GPU per process, made the only visible device before CUDA starts: the library
        # (its own static CUDA runtime) then works on device 0 like torch does
        os.environ["CUDA_VISIBLE_DEVICES"] = ids[local]
        local = 0

    import torch
    import paper_1612_04082_b200 as eb

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    pk = peaks()
    if args.workload == "gmres":
        return gmres_workload(args, eb, torch)
    if args.workload == "stress":
        return stress_workload(args, eb, torch)

    d = workload(args.n)
    n = d["src"].shape[0]
    t = {k: torch.from_numpy(v).cuda() for k, v in d.items() if isinstance(v, np.ndarray)}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tree = eb.fmm_build_tree(t["src"], t["nrm"], t["w"], max_pts=args.max_pts, p=args.p, K=d["K"], G=d["G"])
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0      # includes the one-time operator precompute
    t0 = time.perf_counter()
    tree2 = eb.fmm_build_tree(t["src"], t["nrm"], t["w"], max_pts=args.max_pts, p=args.p, K=d["K"], G=d["G"])
    torch.cuda.synchronize()
    rebuild_cold_s = time.perf_counter() - t0    # operators cached, device blocks newly allocated
    # steady state of a loop that rebuilds the tree after the geometry changed: the previous
    # tree released first, so its device blocks are reused (tree + lists + schedule only)
    rebuild_s = 1e9
    for _ in range(3):
        del tree2                      # fmm_tree_free: the blocks go back to the library's cache
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tree2 = eb.fmm_build_tree(t["src"], t["nrm"], t["w"], max_pts=args.max_pts, p=args.p, K=d["K"], G=d["G"])
        torch.cuda.synchronize()
        rebuild_s = min(rebuild_s, time.perf_counter() - t0)
    del tree2
    info = eb.fmm_tree_info(tree)
    out = torch.empty((n, 3), device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")   # 256 MB > 126 MB L2

    for _ in range(max(args.warmup, 3)):
        eb.fmm_matvec(tree, eb.KERNEL_UP, t["f"], t["g"], out=out)
    torch.cuda.synchronize()

    # ---- timed region: K steps, L2 flushed between steps (flush outside the events)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = eb.ebem_launch_count()
    # in-situ phase times: every timed step brackets each phase with CUDA events on the stream
    # it runs on (the normal overlapped schedule; fmm_set_profiling mode 2)
    eb.fmm_set_profiling(tree, "insitu")
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(smi_index) as clk:
        for k in range(args.steps):
            flush.fill_(float(k))
            ev[k][0].record()
            eb.fmm_matvec(tree, eb.KERNEL_UP, t["f"], t["g"], out=out)
            ev[k][1].record()
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches = (eb.ebem_launch_count() - launches0) // args.steps
    ms_steps = [a.elapsed_time(b) for a, b in ev]
    ms = float(np.mean(ms_steps))
    ms = max_over_ranks(ms, dist)
    # (S2L is not timed separately in situ: its time is inside NEAR's, both on stream B)
    insitu = {p["name"]: (p["ms"] if p["ms"] >= 0 else None) for p in eb.fmm_phase_stats(tree, eb.KERNEL_UP)}

    # ---- solo per-phase device times (phases one after another, 5 L2-flushed steps)
    eb.fmm_set_profiling(tree, True)
    for k in range(5):
        flush.fill_(float(k))
        eb.fmm_matvec(tree, eb.KERNEL_UP, t["f"], t["g"], out=out)
    phases = eb.fmm_phase_stats(tree, eb.KERNEL_UP)
    eb.fmm_set_profiling(tree, False)
    ph_out = []
    tensor_phases = ("Q2Z_up", "M2M", "Q2Z_dn", "M2L", "L2L")   # tcgen05 path, three products per fp32 product
    pk["tf32x3_tflops"] = pk["tf32_tflops"] / 3.0                # fp32-equivalent peak of 3xTF32
    pk["f16x3_tflops"] = pk["bf16_tflops"] / 3.0                 # ... of 3xFP16 (fp16 dense = bf16 dense rate)
    # operand type of the M2L (the library's default: FP16 head / remainder, EBEM_M2L_F16 = 0: TF32)
    m2l_f16 = int(os.environ.get("EBEM_M2L_F16", "2")) >= 1
    # at p <= 6 the M2M / L2L chains and the upward Q2Z run on FP16 operands too (library defaults)
    f16_phases = {"M2L"} if m2l_f16 else set()
    if m2l_f16 and args.p <= 6:
        if os.environ.get("EBEM_ML_F16", "1") != "0":
            f16_phases |= {"M2M", "L2L"}
        if os.environ.get("EBEM_Q2Z_F16", "1") != "0":
            f16_phases |= {"Q2Z_up"}
    def tensor_peak(name):
        return pk["f16x3_tflops"] if name in f16_phases else pk["tf32x3_tflops"]
    for ph in phases:
        f64, f32 = ph["flops_fp64"], ph["flops"] - ph["flops_fp64"]
        sec = ph["ms"] * 1e-3
        tmem = ph["bytes"] / (pk["hbm_gbs"] * 1e9)
        if ph["name"] in tensor_phases:
            tmin, bound = ph["flops"] / (tensor_peak(ph["name"]) * 1e12), "tensor"
        else:
            tmin, bound = f32 / (pk["fp32_tflops"] * 1e12) + f64 / (pk["fp64_tflops"] * 1e12), "alu"
        if tmem > tmin:
            bound = "hbm"
        frac = (max(tmin, tmem) / sec) if sec > 0 else None
        isec = (insitu.get(ph["name"]) or 0) * 1e-3
        ph_out.append({"name": ph["name"], "ms": ph["ms"], "ms_in_situ": insitu.get(ph["name"]),
                       "launches": ph["launches"], "bound": bound,
                       "gflop": ph["flops"] / 1e9, "gflop_fp64": f64 / 1e9, "interactions": ph["interactions"],
                       "mbytes": ph["bytes"] / 1e6, "frac": frac,
                       "operands": ("fp16" if ph["name"] in f16_phases else "tf32") if ph["name"] in tensor_phases else None,
                       "frac_in_situ": (max(tmin, tmem) / isec) if isec > 0 else None})
    # dominant kernel: the phase with the most device time (solo; M2L at p = 6), its fraction
    # taken from its in-situ time inside the timed region (M2L and NEAR share the SMs there)
    dom = max(ph_out, key=lambda x: x["ms"] or 0)
    dph = next(p for p in phases if p["name"] == dom["name"])
    sec = (dom["ms_in_situ"] or dom["ms"]) * 1e-3   # in situ: inside the timed, overlapped step
    sec_solo = dom["ms"] * 1e-3
    if dom["bound"] == "tensor":
        tpk = tensor_peak(dom["name"])
        f16 = dom["name"] == "M2L" and m2l_f16
        roof = {"bound": "tensor", "phase": dom["name"], "achieved": dph["flops"] / sec / 1e12,
                "peak": tpk, "unit": "TFLOP/s", "frac": dph["flops"] / sec / 1e12 / tpk,
                "frac_in_situ": dph["flops"] / sec / 1e12 / tpk,
                "frac_solo": dph["flops"] / sec_solo / 1e12 / tpk,
                "ms_in_situ": dom["ms_in_situ"], "ms_solo": dom["ms"], "traffic": None,
                "operands": "fp16 head/remainder (3xFP16)" if f16 else "tf32 head/remainder (3xTF32)",
                "peak_source": ("measured bf16 GEMM (fp16 dense = bf16 dense rate) / 3 (3xFP16 = fp32-accurate)" if f16 else
                                "measured bf16 GEMM x 1.1/2.25 (guide's nominal TF32 / bf16 dense ratio) / 3 "
                                "(3xTF32 = fp32-accurate)") +
                               "; achieved counts algorithmic fp32 flops 2*M*K per pair; "
                               "frac = frac_in_situ (CUDA events on the M2L stream inside the timed region), "
                               "frac_solo = the phase run alone (incl. the fp16 split of the Z rows)"}
        if f16:   # the same time against the round-1 denominator (3xTF32), for comparison across rounds
            roof["frac_solo_vs_tf32x3_peak"] = dph["flops"] / sec_solo / 1e12 / pk["tf32x3_tflops"]
    elif dom["bound"] == "alu":
        f64, f32 = dph["flops_fp64"], dph["flops"] - dph["flops_fp64"]
        peak = dph["flops"] / (f32 / pk["fp32_tflops"] + f64 / pk["fp64_tflops"]) if dph["flops"] else pk["fp32_tflops"]
        roof = {"bound": "alu", "phase": dom["name"], "achieved": dph["flops"] / sec / 1e12, "peak": peak,
                "unit": "TFLOP/s", "frac": dph["flops"] / sec / 1e12 / peak,
                "frac_in_situ": dph["flops"] / sec / 1e12 / peak, "frac_solo": dph["flops"] / sec_solo / 1e12 / peak,
                "ms_in_situ": dom["ms_in_situ"], "ms_solo": dom["ms"], "traffic": None,
                "peak_source": f"derived: 148 SM x 128 FP32 (64 FP64) lanes x 2 x {pk['fp32_tflops']/148/256*1e6:.0f} MHz"
                               "; achieved counts the pair loop's FP32 flops (FFMA = 2, counted in SASS); "
                               "frac = frac_in_situ (CUDA events on the kernel's stream inside the timed region, "
                               "where it shares the SMs with the M2L), frac_solo = the phase run alone"}
        # the other large kernel of the overlapped region, for reference
        m2l = next((p for p in ph_out if p["name"] == "M2L"), None)
        if m2l and dom["name"] != "M2L":
            roof["m2l"] = {"ms_solo": m2l["ms"], "ms_in_situ": m2l["ms_in_situ"], "frac_solo": m2l["frac"],
                           "frac_in_situ": m2l["frac_in_situ"], "peak": tensor_peak("M2L"), "unit": "TFLOP/s",
                           "operands": "fp16 head/remainder (3xFP16)" if m2l_f16 else "tf32 head/remainder (3xTF32)"}
    else:
        roof = {"bound": "hbm", "phase": dom["name"], "achieved": dph["bytes"] / sec / 1e9, "peak": pk["hbm_gbs"],
                "unit": "GB/s", "frac": dph["bytes"] / sec / 1e9 / pk["hbm_gbs"], "traffic": None,
                "peak_source": pk["src"]}

    # DRAM traffic of the dominant kernel: dram__bytes_read.sum + dram__bytes_write.sum per launch
    # from the committed ncu --set full capture of this round (profiles/r02/traffic.json names
    # the capture file and the row it was read from)
    for rnd in ("r02", "r01"):
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", rnd, "traffic.json")))
        except Exception:
            continue
        if roof["phase"] in tr:
            rec = tr[roof["phase"]]
            roof["traffic"] = rec["dram_read"] + rec["dram_write"]
            roof["traffic_source"] = rec.get("source") or tr.get("_source")
            roof["traffic_vs_algorithmic"] = roof["traffic"] / max(dph["bytes"], 1.0)
            break

    # ---- e2e through the C ABI with host buffers (pinned), copies inside the timed region
    fh = torch.from_numpy(d["f"]).pin_memory().numpy()
    gh = torch.from_numpy(d["g"]).pin_memory().numpy()
    oh = torch.empty((n, 3), dtype=torch.float32).pin_memory().numpy()
    eb.fmm_matvec(tree, eb.KERNEL_UP, fh, gh, out=oh)
    e2e = []
    for k in range(max(2, args.steps // 2)):
        flush.fill_(float(k))
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eb.fmm_matvec(tree, eb.KERNEL_UP, fh, gh, out=oh)
        b.record()
        torch.cuda.synchronize()
        e2e.append(a.elapsed_time(b))

    p2p = None if args.no_p2p else p2p_bench(eb, torch, pk)

    # ---- CPU oracle on a bounded target sample (rank 0, N = 1 only) + accuracy on it
    cpu = None
    rel = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rng = np.random.default_rng(7)
        idx = np.sort(rng.choice(n, args.cpu_sample, replace=False))
        ref, sec, cores = oracle_sample(d, idx)
        got = out.cpu().numpy().astype(np.float64)[idx]
        rel = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
        cpu = {"value": 1e3 * sec * n / args.cpu_sample, "unit": "ms", "cores": cores, "kind": "oracle",
               "sample": f"{args.cpu_sample} random targets x all {n} sources (fp64 C direct sum), "
                         f"{sec:.1f} s, extrapolated to all {n} targets"}

    # ---- configs[2]'s second order: the same points at p = 10 (fp64 far field, drained
    # tensor-core accumulation), 5 L2-flushed steps, error on the same oracle sample
    p10 = None
    if rank == 0 and world == 1 and not args.no_p10 and args.p != 10:
        tree10 = eb.fmm_build_tree(t["src"], t["nrm"], t["w"], max_pts=args.max_pts, p=10, K=d["K"], G=d["G"])
        out10 = torch.empty_like(out)
        for _ in range(2):
            eb.fmm_matvec(tree10, eb.KERNEL_UP, t["f"], t["g"], out=out10)
        ts = []
        for k in range(5):
            flush.fill_(float(k))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            eb.fmm_matvec(tree10, eb.KERNEL_UP, t["f"], t["g"], out=out10)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        p10 = {"p": 10, "ms": float(np.mean(ts)), "steps": 5, "rel_l2": None}
        if rel is not None:
            got10 = out10.cpu().numpy().astype(np.float64)[idx]
            p10["rel_l2"] = float(np.linalg.norm(got10 - ref) / np.linalg.norm(ref))
        del tree10

    # ---- configs[3] (stress evaluation) and configs[4] (GMRES solve)
    stress = gmres = gmres_paper = None
    if rank == 0 and world == 1:
        del tree
        torch.cuda.empty_cache()
        if not args.no_stress:
            stress = stress_workload(args, eb, torch, emit=False)
        if not args.no_gmres:
            gmres = gmres_workload(args, eb, torch, emit=False, precond=2)
        if not args.no_gmres_paper:      # plain restarted GMRES, no preconditioner
            args.max_iter = max(args.max_iter, 3000)
            gmres_paper = gmres_workload(args, eb, torch, emit=False, precond=0)

    if rank == 0:
        line = {"metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32 (3xFP16 tensor-core translations; fp64 plan, fp64 equivalent densities)",
                "data": "synthetic",
                "config": {"workload": WORKLOAD, "n_points": n, "p": args.p, "max_pts": args.max_pts,
                           "kernel": "UP", "l2": "flushed between steps (256 MB write)",
                           "nboxes": info["nboxes"], "nlevels": info["nlevels"], "n_v": info["n_v"],
                           "parallelism": "replicas" if world > 1 else "single"},
                "points_per_s": world * n / (ms * 1e-3), "rel_l2": rel, "tree_build_s": rebuild_s,
                "tree_build_cold_blocks_s": rebuild_cold_s,
                "first_build_s_incl_operators": build_s, "gpu_launches": int(launches),
                "roofline": roof, "phases": ph_out, "p2p": p2p, "p10": p10, "stress": stress, "gmres": gmres,
                "gmres_paper": gmres_paper,
                "cpu_baseline": cpu,
                "e2e": {"value": float(np.mean(e2e)), "unit": "ms", "h2d_bytes_per_step": int(fh.nbytes + gh.nbytes),
                        "d2h_bytes_per_step": int(oh.nbytes)},
                "clocks": clk.summary(), "peaks": pk}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
