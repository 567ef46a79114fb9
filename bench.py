#!/usr/bin/env python
"""Benchmark of the B200 H² factorize + solve hot path (BASELINE.json metric:
"H² factorization unknowns/s & FP64 TFLOP/s vs peak; solve time; rel. residual").

One step = factorize (the level-by-level H² LU) + one solve of a seeded
complex-normal right-hand side, on BASELINE config 2 by default (VIE
dielectric cube 32^3 = 32768 unknowns, leaf 32, eta 1, eps 1e-4, complex128).
The H² input is built on the GPU once, outside the timed region.

  value  unknowns/s of the factorization, device time (CUDA events on the
         library stream), inputs resident in HBM, max over ranks
  e2e    same metric through the public C-ABI calls with HOST buffers: every
         step uploads the H² matrix (h2g_matrix_upload) and the RHS from host
         memory, builds the symbolic plan from scratch (cold structure),
         factorizes, solves and reads x back (wall clock around the
         synchronous calls, max over ranks); e2e.warm reuses the plan

Multi-GPU (--gpus N under torch.distributed.run, N in {2, 4, 8}): ONE
factorization partitioned over the ranks (h2g.factorize_dist: the 8 level-3
subtrees are dealt to the ranks, interior clusters eliminated locally, one
NCCL exchange per level, boundary clusters and coarse levels replicated;
DESIGN.md §7). Total work is fixed, so scaling is "strong" and `value` is
N_unknowns / max-over-ranks time. --impl reference times the CPU restatement
of the reference (oracle/, the reference itself cannot be built here: Eigen is
absent) on rank 0 only.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------- helpers
def load_peaks():
    peaks = {}
    try:
        peaks.update(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))))
    except Exception:
        pass
    try:
        peaks.update(json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json"))))
    except Exception:
        pass
    return peaks


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_threads():
    """Threads the oracle's worker pool uses (H2O_THREADS, default all cores)."""
    v = os.environ.get("H2O_THREADS")
    return max(1, int(v)) if v else (os.cpu_count() or 1)


def golden_cpu_reference(config):
    """The full-config oracle factorization measured once (tests/golden,
    written by scripts/oracle_golden.py), if committed for this config."""
    f = os.path.join(ROOT, "tests", "golden", f"cfg{config}_oracle.json")
    if not os.path.exists(f):
        return None
    try:
        g = json.load(open(f))
    except Exception:
        return None
    return {"value": g["n"] / g["oracle_factor_s"], "unit": "unknowns/s", "factor_s": g["oracle_factor_s"], "cores": g["oracle_threads"],
            "nproc": g["nproc"], "cpu_model": g["cpu_model"], "when": g["when"], "source": os.path.relpath(f, ROOT),
            "note": f"oracle factorization of the full BASELINE config {config} (N={g['n']}) measured once on the GPU box host"}


def cpu_oracle_sample():
    """Bounded CPU sample of the config-2 workload: the oracle (CPU
    restatement of the reference, reference order) factorizing one octant of
    the config-2 cube, i.e. the 16^3 sub-cube at the same spacing h = 1/32,
    leaf 32, eps 1e-4 (identical to BASELINE config 1, the reference's own
    CPU-runnable case)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as O
    from paper_1703_06155_b200.geometry import BASELINE_CONFIGS, vie_constants, vie_grid_points

    c = BASELINE_CONFIGS[1]
    k0, scale, diag = vie_constants(c["cells"], c["side"])
    t = O.Tree(vie_grid_points(c["cells"], c["side"]), c["leaf"])
    A = O.H2(O.Blocks(t, 1.0), O.helmholtz(k0, diag, scale), c["eps"])
    return A, c, O


SAMPLE_NOTE = ("oracle/ (CPU restatement of proj/include/h2lu/factorization.hpp, reference cluster order; independent block "
               "products on a worker pool, bit-identical to 1 thread) factorizing one octant of the config-2 cube per step: the "
               "16^3 sub-cube at the same h = 1/32, leaf 32, eps 1e-4 (= BASELINE config 1, N=4096). unknowns/s on the octant "
               "overstates the CPU's full-cube rate (work per unknown grows with N); the full config-2 oracle run measured once "
               "is under full_config")


def workload_config(config, schedule="reference", world=1):
    from paper_1703_06155_b200.geometry import BASELINE_CONFIGS

    c = BASELINE_CONFIGS[config]
    n = c["cells"] ** 3
    return {"workload": f"BASELINE config {config}: VIE dielectric cube {c['cells']}^3 = {n} unknowns, side {c['side']} lambda, eps_r 4, "
                        f"leaf {c['leaf']}, eta 1, eps_h2 = eps_fill = {c['eps']}",
            "n": n, "schedule": schedule if world == 1 else "subtree",
            "parallelism": (f"subtree partition x{world}: level-3 subtrees dealt to the ranks, interior clusters local, one exchange per level, "
                            "boundary clusters and coarse levels replicated") if world > 1 else "1 GPU",
            "l2": "inputs larger than L2 (dense leaf blocks alone exceed 126 MB)"}


def run_reference(args, rank):
    if rank != 0:
        return None
    A, c, O = cpu_oracle_sample()
    n = A.n
    for _ in range(args.warmup):
        A.factorize(c["eps"])
    secs = []
    for _ in range(args.steps):
        ch = A.factorize(c["eps"])
        secs.append(ch.seconds)
    t = float(np.mean(secs))
    value = n / t
    cpu = {"value": value, "unit": "unknowns/s", "cores": oracle_threads(), "nproc": os.cpu_count(), "cpu_model": cpu_model(), "kind": "port",
           "sample": SAMPLE_NOTE, "full_config": golden_cpu_reference(args.config)}
    return {
        "metric": "H2 factorization unknowns/s",
        "value": value,
        "unit": "unknowns/s",
        "impl": "reference",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "complex128",
        "data": "synthetic",
        "config": workload_config(args.config, args.schedule, args.gpus),
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": "unknowns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# --------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--schedule", default="reference", choices=["reference", "colored"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist

        # one GPU per rank: NCCL over NVLink; ranks sharing a GPU (single-GPU test boxes) or no GPU (reference arm on CPU): gloo
        ndev = torch.cuda.device_count() if torch.cuda.is_available() else 0
        backend = "nccl" if ndev >= world else "gloo"
        if ndev:
            local = local % ndev
            torch.cuda.set_device(local)
        dist.init_process_group(backend)

    if args.impl == "reference":
        out = run_reference(args, rank)
        if out is not None:
            print(json.dumps(out), flush=True)
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    import paper_1703_06155_b200 as h2g
    from paper_1703_06155_b200.geometry import BASELINE_CONFIGS, vie_constants, vie_grid_points

    c = BASELINE_CONFIGS[args.config]
    eps = c["eps"]
    k0, scale, diag = vie_constants(c["cells"], c["side"])
    pts = vie_grid_points(c["cells"], c["side"])
    n = pts.shape[0]
    ctx = h2g.Context(local)
    t0 = time.perf_counter()
    A = h2g.H2Matrix.build(pts, c["leaf"], 1.0, h2g.helmholtz_kernel(k0, diag, scale), eps, ctx)
    build_s = time.perf_counter() - t0
    host = A.download()
    perm = host["perm"]
    b = h2g.random_rhs(n, 1234)[perm]  # seeded, original order -> tree order
    log(f"[bench] rank {rank}: built H2 for N={n} in {build_s:.2f}s")

    def sync_all():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(v):
        if dist is None:
            return v
        import torch

        t = torch.tensor([v], dtype=torch.float64, device=f"cuda:{local}" if torch.cuda.is_available() else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def fact(M):
        # N > 1: one factorization partitioned over the ranks (strong scaling)
        if world > 1:
            return h2g.factorize_dist(M, eps)
        return h2g.factorize(M, eps, schedule=args.schedule)

    for _ in range(args.warmup):
        ch = fact(A)
        x = ch.solve(b)
        del ch
    sync_all()
    sampler = ClockSampler(local)
    sampler.start()
    fms, sms, flaunch, slaunch = [], [], [], []
    ch = None
    for _ in range(args.steps):
        ch = None  # release the previous chain first: its device blocks are reused
        ch = fact(A)
        x = ch.solve(b)
        tm = ch.timing()
        fms.append(tm["factor_ms"])
        sms.append(tm["solve_ms"])
        flaunch.append(tm["factor_launches"])
        slaunch.append(tm["solve_launches"])
    clocks = sampler.stop()
    sync_all()
    factor_ms = max_over_ranks(float(np.mean(fms)))
    solve_ms = max_over_ranks(float(np.mean(sms)))
    work = ch.work()
    ranks = [r["rank_after"] for r in ch.all_records()]
    levels = ch.levels()
    residual = A.relative_residual(x, b)
    pts_tree = pts[perm]
    rows = np.sort(np.random.default_rng(1234).choice(n, size=min(4096, n), replace=False)).astype(np.int64)
    sampled = h2g.sampled_dense_residual(pts_tree, h2g.helmholtz_kernel(k0, diag, scale), x, b, rows, ctx)
    # cold symbolic plan: the first factorize of a new structure builds it on
    # the host (outside the device factor time); later ones reuse it
    ctx.clear_plans()
    Acold = h2g.H2Matrix.upload(host, ctx)
    chc = fact(Acold)
    plan_cold_ms = max_over_ranks(chc.timing()["plan_ms"])
    del chc, Acold

    # ---- end to end through the C ABI with host buffers
    e2e = None
    if not args.no_e2e:
        h2d = sum(v.nbytes for k, v in host.items() if isinstance(v, np.ndarray)) + b.nbytes
        d2h = x.nbytes
        try:
            import torch

            cudart = torch.cuda.cudart()
            for v in list(host.values()) + [b]:
                if isinstance(v, np.ndarray) and v.nbytes:
                    cudart.cudaHostRegister(v.ctypes.data, v.nbytes, 0)
            pinned = True
        except Exception:
            pinned = False
        def e2e_run(cold):
            ts, plan = [], []
            for i in range(1 + args.steps):
                if cold:
                    ctx.clear_plans()  # new structure every step: the host plan is built inside the timed region
                t0 = time.perf_counter()
                G = h2g.H2Matrix.upload(host, ctx)
                ch2 = fact(G)
                x2 = ch2.solve(b)
                t1 = time.perf_counter()
                plan.append(ch2.timing()["plan_ms"])
                del ch2, G
                if i >= 1:
                    ts.append(t1 - t0)
            sync_all()
            return max_over_ranks(float(np.mean(ts))), float(np.mean(plan[1:])), x2

        te2e, plan_e2e, x2 = e2e_run(cold=True)
        twarm, plan_warm, _ = e2e_run(cold=False)
        e2e = {"value": n / te2e, "unit": "unknowns/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "s_per_step": te2e, "plan_ms_per_step": plan_e2e, "pinned_host": pinned,
               "timing": "wall clock around synchronous C-ABI calls (upload from pinned host memory, symbolic plan built from scratch, "
                         "factorize, solve, x read back), max over ranks",
               "solution_matches_resident_run": bool(np.allclose(x2, x, rtol=0, atol=1e-12 * np.abs(x).max())),
               "warm": {"value": n / twarm, "s_per_step": twarm, "plan_ms_per_step": plan_warm,
                        "note": "same, with the symbolic plan reused from the context's structure-keyed cache (refactorization of the "
                                "same geometry with new entries)"}}

    # ---- roofline of the dominant kernel class (separate profiled run)
    ctx.set_profiling(True)
    chp = fact(A)
    ctx.set_profiling(False)
    dstats = ch.dist_stats() if world > 1 else None
    # the colored order (one colour per batch: ~150 batches instead of ~1250 wavefronts) as a second data point
    other = None
    if world == 1 and args.schedule == "reference":
        chq = h2g.factorize(A, eps, schedule="colored")
        del chq
        chq = h2g.factorize(A, eps, schedule="colored")
        xq = chq.solve(b)
        other = {"colored": {"factor_ms": chq.timing()["factor_ms"], "solve_ms": chq.timing()["solve_ms"],
                             "relative_residual_h2": A.relative_residual(xq, b),
                             "note": "greedy distance-1 colouring, one colour per batch (a different valid elimination order; "
                                     "parity-tested against the oracle run in that order)"}}
        del chq
    # 64 right-hand sides through the explicit-inverse application (config 4's mode), outside the timed region
    many = None
    if world == 1:
        B64 = np.stack([h2g.random_rhs(n, 1234 + j) for j in range(64)], axis=1)[perm]
        ms64 = []
        for _ in range(3):
            X64 = ch.apply_inverse_explicit(B64)
            ms64.append(ch.timing()["solve_ms"])
        many = {"nrhs": 64, "mode": "apply_inverse_explicit", "ms": min(ms64),
                "relative_residual_h2_col63": A.relative_residual(X64[:, 63], B64[:, 63]),
                "note": "right-hand-side groups side by side in one launch per level and direction (best of 3)"}
        del B64, X64
    stats = chp.kernel_stats()
    prof_total = sum(v["ms"] for v in stats.values())
    dom = max(stats, key=lambda k: stats[k]["ms"])
    peaks = load_peaks()
    peak_tf = peaks.get("zgemm_tflops")
    peak_src = "measured cuBLAS ZGEMM 4096^3 on this pool (profiles/fp64_peak.json)"
    if not peak_tf:
        peak_tf, peak_src = 37.0, "fallback: nominal B200 FP64 ~37 TFLOP/s (no measured FP64 peak found)"
    hbm = peaks.get("hbm_gbs", 6469.3)
    sch = stats["schur"]
    roof = None
    if sch["ms"] > 0:
        t_s = sch["ms"] / 1e3
        exw = chp.work()
        ex_flops, ex_bytes = exw["schur_flops_executed"], exw["schur_bytes_executed"]
        tf = ex_flops / t_s / 1e12
        gbs = ex_bytes / t_s / 1e9
        nl = max(sch["launches"], 1)
        if ex_flops / (peak_tf * 1e12) >= ex_bytes / (hbm * 1e9):
            roof = {"kernel": "k_schur (step 3c Schur scatter)", "bound": "tensor", "achieved": tf, "peak": peak_tf, "unit": "TFLOP/s",
                    "frac": tf / peak_tf, "peak_source": peak_src + " (FP64 has no tcgen05 path; DMMA/DFMA peak)"}
        else:
            roof = {"kernel": "k_schur (step 3c Schur scatter)", "bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
        traffic, tsrc, alone = None, None, None
        import glob
        for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_schur_traffic.json"))):
            try:
                tj = json.load(open(f))
            except Exception:
                continue
            if tj.get("config") == args.config and tj.get("launches") == sch["launches"]:
                traffic, tsrc = tj["traffic_per_launch"], os.path.relpath(f, ROOT) + " (ncu dram__bytes_read+write per k_schur launch, same launch list)"
                if tj.get("serialised_ms"):
                    # not a live number: the committed ncu launch list, every k_schur launch alone on the GPU (no overlap with the
                    # chain kernels of the other stream, cold caches); explains the gap to the live event time above
                    alone = {"ms": tj["serialised_ms"], "tflops": ex_flops / (tj["serialised_ms"] / 1e3) / 1e12,
                             "frac": ex_flops / (tj["serialised_ms"] / 1e3) / 1e12 / peak_tf, "source": os.path.relpath(f, ROOT),
                             "note": "profiler-derived (ncu gpu__time_duration.sum summed over the launches of one factorize), not measured in this run"}
        roof.update({"basis": "executed work: the products k_schur computes (rows/columns of clusters eliminated in an earlier batch "
                              "are exact zeros and are skipped, factorization.hpp:431-439); flops_per_launch x launches / k_schur event time",
                     "flops_per_launch": ex_flops / nl, "bytes_per_launch": ex_bytes / nl,
                     "traffic": traffic, "traffic_source": tsrc, "kernel_alone": alone, "launches": sch["launches"], "avg_launch_us": 1e3 * sch["ms"] / nl,
                     "share_of_factorize": sch["ms"] / max(prof_total, 1e-9),
                     "algorithmic": {"flops": sch["flops"], "tflops": sch["flops"] / t_s / 1e12, "frac": sch["flops"] / t_s / 1e12 / peak_tf,
                                     "note": "SURVEY 8d count (full b_j x e x b_c products, as the reference's GEMMs execute them, "
                                             "including the exact-zero rows/columns k_schur skips)"}})
        # per level: a launch is bound by whichever of its flops / bytes takes longer at peak
        # (fine levels: e of a few columns, the target read-modify-write dominates -> HBM)
        per_level, bound_ms = [], 0.0
        for lv in chp.schur_levels():
            if lv["ms"] <= 0:
                continue
            t_f, t_b = lv["flops"] / (peak_tf * 1e12), lv["bytes"] / (hbm * 1e9)
            bound_ms += 1e3 * max(t_f, t_b)
            per_level.append({"level": lv["level"], "ms": round(lv["ms"], 2), "tflops": round(lv["flops"] / lv["ms"] / 1e9, 2),
                              "gbs": round(lv["bytes"] / lv["ms"] / 1e6, 1), "bound": "tensor" if t_f >= t_b else "hbm",
                              "frac": round(1e3 * max(t_f, t_b) / lv["ms"], 3)})
        roof["per_level"] = per_level
        roof["per_level_note"] = ("executed flops / algorithmic bytes (targets read + written once per launch, panels read once per target) "
                                  "per level against the FP64 and HBM peaks; frac = the larger of the two lower bounds / event time")
        roof["frac_mixed_bound"] = bound_ms / sch["ms"]
    solve_roof = None
    if solve_ms > 0:
        sgbs = work["solve_bytes"] / (solve_ms / 1e3) / 1e9
        solve_roof = {"kernel": "solve (k_fwd_flow / k_bwd_flow dataflow level kernels, nrhs = 1)", "bound": "hbm", "achieved": sgbs, "peak": hbm, "unit": "GB/s",
                      "frac": sgbs / hbm, "bytes": work["solve_bytes"],
                      "basis": "chain bytes (Qtilde read twice, L11/U11/Lbar/Ubar, root triangles) + 4 x 16 x N vector traffic per solve "
                               "/ device solve time"}
    breakdown = {k: {"ms": round(v["ms"], 3), "launches": v["launches"]} for k, v in stats.items()}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        Ao, co, O = cpu_oracle_sample()
        cho = Ao.factorize(co["eps"])
        cpu = {"value": Ao.n / cho.seconds, "unit": "unknowns/s", "cores": oracle_threads(), "nproc": os.cpu_count(), "cpu_model": cpu_model(),
               "kind": "port", "sample": SAMPLE_NOTE + f" (this run: {cho.seconds:.2f} s)", "full_config": golden_cpu_reference(args.config)}

    out = {
        "metric": "H2 factorization unknowns/s",
        "value": n / (factor_ms / 1e3),
        "unit": "unknowns/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": factor_ms + solve_ms,
        "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None,
        "dtype": "complex128",
        "data": "synthetic",
        "config": workload_config(args.config, args.schedule, world),
        "factor_ms": factor_ms,
        "dist": dstats,
        "other_schedules": other,
        "many_rhs": many,
        "plan_ms_cold": plan_cold_ms,
        "factor_ms_incl_cold_plan": factor_ms + plan_cold_ms,
        "solve_ms": solve_ms,
        "factor_tflops": work["factor_flops"] / (factor_ms / 1e3) / 1e12,
        "solve_gbs": work["solve_bytes"] / (solve_ms / 1e3) / 1e9 if solve_ms > 0 else None,
        "relative_residual_h2": residual,
        "relative_residual_sampled_dense": sampled,
        "rank_max": int(max(ranks)) if ranks else 0,
        "root_size": ch.root_size,
        "levels": [{k: lv[k] for k in ("level", "rank_sum_after", "eliminated", "ledger_blocks")} for lv in levels],
        "build_s": build_s,
        "clocks": clocks,
        "e2e": e2e,
        "gpu_launches": int(np.mean(flaunch) + np.mean(slaunch)),
        "roofline": roof,
        "solve_roofline": solve_roof,
        "kernel_breakdown_ms": breakdown,
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
