#!/usr/bin/env python
"""GMT* benchmark (BASELINE.json metric: p50 ms per GMT* solve at n samples;
batched plans/sec at 1/2/4/8 B200).  One JSON line on rank 0.

Headline workload (BASELINE.json configs[4], `--workload di6d_batched`):
4096 random 6D double-integrator queries per step -- each its own forest of
60 AABB pillars extruded over the velocity axes, start and goal, from
Pcg32(mix64(master, q)) -- n = 4000 Halton samples, cost threshold r = 1.6,
lambda = 1.  The queries are sharded over the ranks (strong scaling: rank r
solves shard_range(4096, N, r)); the only collective is the final gather of
one record per query.  Every query's instance is derived on the GPU from the
shared Halton sample pool (csrc/pool.cu) and is
bit-identical to a single build_instance of that problem.

  value      plans/s over all ranks with every query's instance resident in
             HBM (~20 GB per 4096 queries, far above the 126 MB L2): one
             step = one batched solve launch of the rank's queries (CUDA
             events on the library stream, max over ranks)
  e2e        the same metric end to end through gmt_plan_problems: the
             step's problem descriptions (host structs: boxes, goal, init,
             n, sampling, model) in, the instances derived on the device
             (free masks, ranks, goal substitution, init rows, padded rows
             from the pool graph), one batched solve, summaries out; the pool
             graph itself is built once per (sampling source, radius, model)
             and reused across steps (pool_build_ms)
  roofline   HBM roofline of the solve kernel: SURVEY.md §8(d)'s algorithmic
             bytes 12*InScan + 4*OutScan + 8*OpenParentReads + 9*V*Passes
             counted on the device, over one launch's own duration
  cpu_baseline / --impl reference  the unmodified reference gmt_plan
             (oracle/_ref) on the host cores over a 64-query sample of the
             same instances (graphs from the oracle's statement of the DI
             model, cached polylines), parallel_chunks(nproc), plan-only
  parity     the GPU summaries of the sample vs the reference's (status,
             cost bits, iterations, checks)
Secondary legs (configs[1-3]): the 3D forest batch (512 queries), p50 single
solves of the C2 forest, the 6D DI n=4000 instance and the 12D quadrotor.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
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

METRIC = "GMT* plans/sec (batched queries); p50 ms per single solve"
UNIT = "plans/s"
MASTER_SEED = 20171005


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--queries", type=int, default=4096, help="DI queries per step (all ranks together)")
    ap.add_argument("--n", type=int, default=4000)
    ap.add_argument("--radius", type=float, default=1.6)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--single-reps", type=int, default=101)
    ap.add_argument("--ref-reps", type=int, default=21, help="reference single-solve calls per leg")
    ap.add_argument("--cpu-sample", type=int, default=64, help="queries in the CPU baseline sample")
    ap.add_argument("--cpu-threads", type=int, default=0, help="reference threads (0: every host core)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--forest-queries", type=int, default=512,
                    help="configs[1] 3D forest batch per GPU (0: skip the secondary legs)")
    ap.add_argument("--no-quad", action="store_true", help="skip the 12D quadrotor leg (configs[3])")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def di_specs(queries, n: int, radius: float):
    """configs[4]: query q = random_di_query(master, q) (its own forest,
    start and goal from Pcg32(mix64(master, q)))."""
    from paper_1705_02403_b200 import problem as P
    return [P.random_di_query(MASTER_SEED, q, n=n, radius=radius) for q in queries]


def forest_specs(rank: int, per_gpu: int, n: int):
    from paper_1705_02403_b200 import problem as P
    from paper_1705_02403_b200.shard import weak_range
    return [P.random_forest_query(MASTER_SEED, q, n=n) for q in weak_range(per_gpu, rank)]


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.stop = threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)

    def _nvml(self):
        """NVML handle of this rank's GPU (by PCI bus id), or None."""
        try:
            import pynvml
            pynvml.nvmlInit()
            try:
                import torch
                p = torch.cuda.get_device_properties(self.device)
                bus = "%08x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
                return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.device)
        except Exception:
            return None

    def run(self):
        nv = self._nvml()
        if nv is not None:  # NVML: ~1 ms per sample, so short timed regions get many
            pynvml, h = nv
            bits = (pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap)
            while not self.stop.is_set():
                try:
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append([str(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)),
                                      str(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))] +
                                     ["Active" if r & b else "Not Active" for b in bits])
                except Exception:
                    break
                self.stop.wait(0.01)
            if self.rows:
                return
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.05)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def ncu_traffic(kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`
    from the committed ncu --set full summary (profiles/<round>/ncu_summary.json)."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_summary.json")), reverse=True):
        try:
            with open(path) as f:
                d = json.load(f)
            k = d["kernels"][kernel]
            return k["dram_bytes_read"] + k["dram_bytes_write"], os.path.relpath(path, ROOT)
        except Exception:
            continue
    return None, None


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback"


# --------------------------------------------------------------------------
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_threads(args) -> int:
    return args.cpu_threads or os.cpu_count() or 1


def reference_di(specs, threads: int, passes: int, warmup: int = 1):
    """The unmodified reference gmt_plan (oracle/_ref) on DI instances of
    `specs`: the reference's own sample_free + append_init, the graph from
    the oracle's C statement of the DI model over the shared Halton pool,
    cached waypoint polylines; one gmt_plan(workers=1) per query under
    parallel_chunks(threads) (the simulator.cpp:212 pattern), plan-only.
    -> (plans/s per pass, summaries, build seconds)."""
    import oracle
    R = oracle.ref()
    t0 = time.perf_counter()
    from paper_1705_02403_b200.problem import halton_pool_size
    need = halton_pool_size(specs)
    pool = R.di_pool(specs[0].start_index, need, specs[0].di_params(), specs[0].radius_override, threads)
    insts = R.di_instances(pool, specs, threads)
    build_s = time.perf_counter() - t0
    for _ in range(warmup):
        R.plan_many(insts, 1.0, threads)
    secs, summ = [], None
    for _ in range(passes):
        summ, sec = R.plan_many(insts, 1.0, threads)
        secs.append(sec)
    del insts, pool
    return [len(specs) / x for x in secs], summ, build_s


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    import oracle
    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libgmtref.so not built"}))
        return
    threads = cpu_threads(args)
    sample = min(args.cpu_sample, args.queries)
    specs = di_specs(range(sample), args.n, args.radius)
    rates, _, build_s = reference_di(specs, threads, args.steps, warmup=args.warmup)
    total = sum(sample / r for r in rates)
    value = sample * len(rates) / total
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total / len(rates) * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": "di6d_batched (configs[4])", "n": args.n, "dim": 6, "boxes": 60,
                   "radius": args.radius, "lambda": 1.0, "queries_per_step": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "cpu": cpu_model(), "nproc": os.cpu_count(),
                         "sample": f"{sample} of the workload's queries per step, gmt_plan(workers=1) per "
                                   f"query under parallel_chunks({threads}); instances built once "
                                   f"({build_s:.1f} s, untimed)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200(args):
    import numpy as np
    import torch

    from paper_1705_02403_b200 import abi, problem as P
    from paper_1705_02403_b200.native import OPT_BATCH_CLUSTER, OPT_BATCH_THREADS, OPT_COUNTERS, Context, ProblemBatch
    from paper_1705_02403_b200.shard import gather_records, records, shard_range

    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))

    def barrier_sync():
        torch.cuda.synchronize()
        ctx.synchronize()
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    def timed_launches(b, k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k):
            b.launch()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1)

    # ---- configs[4]: this rank's shard of the step's DI queries ------------
    mine = shard_range(args.queries, world, rank)
    specs = di_specs(mine, args.n, args.radius)
    pb = ProblemBatch(specs)
    Q = len(specs)

    # instrumented launch (untimed): the algorithmic traffic of one step
    ctx.set_option(OPT_COUNTERS, 1)
    ctx.counters(reset=True)
    cb, _ = ctx.batch_problems(pb)
    cb.launch()
    cnt = ctx.counters(reset=True)
    ctx.set_option(OPT_COUNTERS, 0)
    csum = cb.summaries()
    cb.close()
    del cb
    pool = ctx.pool_info()
    Vpasses = sum(s.num_stats * (spec.n + 1) for s, spec in zip(csum, specs))
    b_alg = 12 * cnt["in_scan"] + 4 * cnt["out_scan"] + 8 * cnt["open_parent_reads"] + 9 * Vpasses

    # ---- device-resident timed loop -----------------------------------------
    t0 = time.perf_counter()
    batch, bst = ctx.batch_problems(pb)
    ctx.synchronize()
    derive_ms = (time.perf_counter() - t0) * 1e3
    for _ in range(args.warmup):
        batch.launch()
    # (a serving loop reads each step's results; from then on the batch
    # dispatches its queries largest-first)
    batch.summaries()
    barrier_sync()
    launches0 = ctx.launch_count
    with ClockSampler(local) as clk:
        total_ms = timed_launches(batch, args.steps)
        barrier_sync()
    launches = ctx.launch_count - launches0
    total_ms = max_over_ranks(total_ms)
    value = args.queries * args.steps / (total_ms / 1e3)
    solo_ms = statistics.median(timed_launches(batch, 1) for _ in range(5))
    dev = batch.summaries()
    if [(a.status, a.cost, a.iterations) for a in dev] != [(a.status, a.cost, a.iterations) for a in csum]:
        raise SystemExit("device-resident results differ between launches")
    peak, peak_kind = measured_peak_hbm()
    achieved = b_alg / (solo_ms / 1e3) / 1e9
    clocks = clk.summary()
    kname = "gmt_solve_kernel<1,6,0,0,0,0,24>"
    traffic, traffic_src = ncu_traffic(kname + ":di6d_q4096")

    batch.close()
    del batch

    # ---- e2e: problem descriptions in, summaries out (gmt_plan_problems) ----
    # One call at a time, then two calls in flight from two host threads
    # (one context each: its own stream, pool and scratch), so one call's
    # host work and instance derivation overlap the other's solve.
    def e2e_check(res):
        pst, psum, _ = res
        if any(int(x) != 0 for x in pst) or [(a.status, a.cost, a.iterations) for a in psum] != \
                [(a.status, a.cost, a.iterations) for a in dev]:
            raise SystemExit("e2e results differ from the device-resident batch")

    for _ in range(max(1, args.warmup)):
        ctx.plan_problems(pb)
    barrier_sync()
    tp = []
    for _ in range(args.e2e_steps):
        t0 = time.perf_counter()
        res = ctx.plan_problems(pb)
        tp.append(time.perf_counter() - t0)
    e2e_check(res)
    e2e_one = args.queries * args.e2e_steps / max_over_ranks(sum(tp))
    pctx = [ctx, Context(local)]
    pctx[1].plan_problems(pb)  # its pool and scratch
    out = [None, None]

    def calls(i):
        for _ in range(args.e2e_steps):
            out[i] = pctx[i].plan_problems(pb)

    barrier_sync()
    pctx[1].synchronize()
    th = [threading.Thread(target=calls, args=(i,)) for i in range(2)]
    t0 = time.perf_counter()
    for x in th:
        x.start()
    for x in th:
        x.join()
    e2e_two = 2 * args.queries * args.e2e_steps / max_over_ranks(time.perf_counter() - t0)
    for r in out:
        e2e_check(r)
    e2e_value = max(e2e_one, e2e_two)
    import ctypes
    prob_h2d = sum(ctypes.sizeof(abi.Problem) + 16 * s.dim * s.num_boxes + 24 * s.dim for s in specs)
    prob_d2h = Q * (40 + 4)
    stage = ctx.pool_info()["stage_ms"]
    pctx[1].close()

    # ---- gather: one record per query to rank 0 (the only collective) -----
    recs = gather_records(records(dev), device=f"cuda:{local}")

    # ---- secondary legs (one GPU) ------------------------------------------
    secondary = None
    if world == 1 and args.forest_queries > 0:
        secondary = secondary_legs(args, ctx, stream)

    line = None
    if rank == 0:
        cpu, parity = None, None
        if not args.no_cpu and world == 1:  # (the CPU baseline: rank 0 at N = 1 only)
            try:
                import oracle
                if oracle.ref_available():
                    threads = cpu_threads(args)
                    sample = min(args.cpu_sample, Q)
                    rates, rsum, build_s = reference_di(specs[:sample], threads, 3)
                    val = statistics.median(rates)
                    cpu = {"value": val, "unit": UNIT, "cores": threads, "kind": "reference",
                           "cpu": cpu_model(), "nproc": os.cpu_count(),
                           "sample": f"the step's first {sample} queries, median of 3 passes, "
                                     f"gmt_plan(workers=1) per query under parallel_chunks({threads}); "
                                     f"instances (reference sample_free/append_init, DI graph + polylines "
                                     f"from the oracle's model statement) built once in {build_s:.1f} s"}
                    same = sum(1 for a, b in zip(dev[:sample], rsum)
                               if (a.status, np.float64(a.cost).tobytes(), a.iterations, a.total_collision_checks)
                               == (b.status, np.float64(b.cost).tobytes(), b.iterations, b.total_collision_checks))
                    parity = f"{same}/{sample} bitwise (status, cost bits, iterations, checks) vs the reference"
            except Exception as e:  # the baseline must never break the bench line
                cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "di6d_batched (configs[4])", "queries_per_step": args.queries,
                       "queries_per_gpu": Q, "n": args.n, "dim": 6, "boxes": 60, "radius": args.radius,
                       "lambda": 1.0, "parallelism": f"dp{world} (query shards)",
                       "l2": "inputs larger than L2 (per-GPU resident derived instances, ~5 MB per query)",
                       "solved": f"{int((recs[:, 0] == 0).sum())}/{len(recs)} success",
                       "pool": {"points": pool["pool_size"], "edges": pool["edges"],
                                "build_ms": pool["build_ms"]},
                       "derive_ms": derive_ms},
            "parity": parity,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": prob_h2d,
                    "d2h_bytes_per_step": prob_d2h,
                    "path": "gmt_plan_problems: problem descriptions in (host), per-query instances derived "
                            "on the device as views of the shared pool (rank maps, special rows), batched solve, "
                            "summaries out",
                    "steps": args.e2e_steps, "one_call_at_a_time": e2e_one, "two_host_threads": e2e_two,
                    "calls_in_flight": 2 if e2e_two > e2e_one else 1},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_kind": peak_kind, "kernel": kname, "bytes_per_launch": b_alg,
                         "kernel_ms": solo_ms,
                         "kernel_ms_note": "one launch alone (CUDA events on the library stream)",
                         "counts": {**cnt, "checks": sum(s.total_collision_checks for s in csum),
                                    "V_passes": Vpasses}},
            "cpu_baseline": cpu,
            "clocks": clocks,
            "gpu_launches": launches,
            "secondary": secondary,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return line


def secondary_legs(args, ctx, stream):
    """configs[0-3] on one GPU: the 3D forest batch; single-solve p50s with
    the reference's single solve on the same instance beside each."""
    import numpy as np
    import torch
    from paper_1705_02403_b200 import problem as P
    from paper_1705_02403_b200.native import OPT_BATCH_CLUSTER, OPT_BATCH_THREADS, ProblemBatch

    out = {}
    specs = forest_specs(0, args.forest_queries, args.n)
    insts = [ctx.build_instance(s) for s in specs]
    b = ctx.batch(insts, 1.0)
    for _ in range(3):
        b.launch()
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(10):
        b.launch()
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    pbf = ProblemBatch(specs)
    ctx.plan_problems(pbf)
    t0 = time.perf_counter()
    for _ in range(5):
        ctx.plan_problems(pbf)
    e2e = len(specs) * 5 / (time.perf_counter() - t0)
    out["forest3d_batched"] = {"workload": "configs[1] 3D forest, 60 pillars, n=4000, formula r",
                               "queries": len(specs), "plans_per_s": len(specs) / ms * 1e3, "ms_per_launch": ms,
                               "e2e_plans_per_s": e2e}
    b.close()
    del insts

    def single_p50(inst):
        res = {}
        for cs in (8, 16):
            ctx.set_option(OPT_BATCH_CLUSTER, cs)
            ctx.set_option(OPT_BATCH_THREADS, 0)
            b1 = ctx.batch([inst], 1.0)
            ctx.set_option(OPT_BATCH_CLUSTER, 0)
            for _ in range(5):
                b1.launch()
            ctx.synchronize()
            times = []
            for _ in range(args.single_reps):
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                b1.launch()
                a1.record(stream)
                a1.synchronize()
                times.append(a0.elapsed_time(a1))
            res[f"cluster{cs}"] = statistics.median(times)
            b1.close()
        return res

    # The reference's single solve on the identical instance (SURVEY.md
    # 8(d)(i)): gmt_plan(workers=1) and (workers=every core), median of
    # --ref-reps calls each timed in C on the monotonic clock.
    R, threads = None, cpu_threads(args)
    if not args.no_cpu:
        import oracle
        R = oracle.ref() if oracle.ref_available() else None

    def ref_single(time_fn):
        if R is None:
            return None
        time_fn(1, 1)  # warm-up
        w1 = float(np.median(time_fn(1, args.ref_reps)))
        wn = float(np.median(time_fn(threads, args.ref_reps)))
        return {"p50_ms_workers1": w1, f"p50_ms_workers{threads}": wn, "reps": args.ref_reps,
                "kind": "reference (oracle/_ref gmt_plan)"}

    def leg(name, spec, inst, ref_fn, **extra):
        s = single_p50(inst)
        r = ctx.plan(inst)
        out[name] = {"p50_ms": min(s.values()), "by_cluster": s, "n": inst.n, "status": r.status,
                     "cost": r.cost, "iterations": r.iterations, **extra}
        rs = ref_single(ref_fn)
        if rs is not None:
            out[name]["reference_single"] = rs
            out[name]["speedup_vs_workers1"] = rs["p50_ms_workers1"] / out[name]["p50_ms"]

    with open(os.path.join(ROOT, "tests", "golden", "scene_texts.json")) as f:
        c0 = P.parse_problem(json.load(f)["rectangles_2d"]).with_n(2000)
    ri0 = R.instance_build(c0, threads) if R else None
    leg("rect2d_single (configs[0])", c0, ctx.build_instance(c0),
        lambda w, k: ri0.time_plans(c0.lam, w, k))
    c1 = P.forest_3d(3, args.n)
    ri1 = R.instance_build(c1, threads) if R else None
    leg("c2_forest_single (configs[1])", c1, ctx.build_instance(c1),
        lambda w, k: ri1.time_plans(1.0, w, k))
    t0 = time.perf_counter()
    c2 = P.di_forest(3, args.n)
    inst2 = ctx.build_instance(c2)
    ctx.synchronize()
    build_ms = (time.perf_counter() - t0) * 1e3
    ri2 = None
    if R:
        from paper_1705_02403_b200.problem import halton_pool_size
        pool = R.di_pool(c2.start_index, halton_pool_size([c2]), c2.di_params(), c2.radius_override, threads)
        [ri2] = R.di_instances(pool, [c2], 1)
    leg("di6d_single (configs[2])", c2, inst2, lambda w, k: ri2.time_plans(1.0, w, k),
        device_build_ms=build_ms, mean_out_degree=inst2.num_edges / inst2.n)
    if not args.no_quad:
        c3 = P.quad_scene()
        t0 = time.perf_counter()
        inst3 = ctx.build_instance(c3)
        ctx.synchronize()
        build_ms = (time.perf_counter() - t0) * 1e3
        fn3 = None
        if R:
            coords, gidx, _ = inst3.download()
            G3 = ctx.build_quad_graph(coords, c3.quad_params(), c3.radius_override, paths=True)
            fn3 = lambda w, k: R.time_gmt_plan(c3, coords, len(gidx), G3, inst3.init_index, 1.0,  # noqa: E731
                                               c3.radius_override, w, k)
        leg("quad12d_single (configs[3])", c3, inst3, fn3, device_build_ms=build_ms)
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
