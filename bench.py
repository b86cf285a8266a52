#!/usr/bin/env python
"""GMT* benchmark (BASELINE.json metric: p50 ms per GMT* solve at n samples;
batched plans/sec at 1/2/4/8 B200).

One JSON line on rank 0.

Workload (BASELINE.json configs[1]): 3D forest of 60 AABB pillars, n=4000
Halton samples, Euclidean cost, formula radius, lambda=1.  A step is one
launch that solves a batch of `--queries` independent queries per GPU (each
query its own forest/start/goal drawn from Pcg32(mix64(master, q)); scenes,
samples and graphs are built on the GPU before timing and stay resident in
HBM: 512 queries x ~6.5 MB of CSR = 3.3 GB per GPU, far above the 126 MB L2,
so no step reads a graph another step left in L2).

  value      plans/s over all ranks, device-resident inputs (CUDA events on
             the library stream, max over ranks)
  e2e        the same metric end to end from problem descriptions through
             gmt_plan_problems: the step's scenes (boxes, goal, init, n,
             sampling) go in from the host, the whole offline phase (sampling,
             init append, r-disk graphs) and the batched solve run on the
             device inside the timed region, summaries come back
  e2e_host_graphs  the same through the C ABI drop-in gmt_plan_batch_host:
             host-resident (pinned) samples + CSR graphs copied H2D, solved,
             summaries + paths + full trees copied D2H (PCIe-bound)
  p50        single-query latency of the canonical C2 instance (Pcg32(3)
             forest) on a cluster of CTAs, p50 over --single-reps launches
  roofline   HBM roofline of the solve kernel with SURVEY.md §8(d)'s
             algorithmic bytes 12*InScan + 4*OutScan + 8*OpenParentReads +
             9*V*Passes counted on the device
  cpu_baseline  the unmodified reference gmt_plan (oracle/_ref) on the
             host cores over a bounded sample of the same queries

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
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--queries", type=int, default=512, help="queries per GPU per step")
    ap.add_argument("--n", type=int, default=4000)
    ap.add_argument("--inflight", type=int, default=2,
                    help="batches in flight: step k+1 is launched on the next stream while step k's slowest "
                         "queries finish (1 = one stream, each step waits for the previous)")
    ap.add_argument("--single-reps", type=int, default=101)
    ap.add_argument("--cpu-sample", type=int, default=64, help="queries in the CPU baseline sample")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--di-queries", type=int, default=296,
                    help="batched 6D double-integrator queries per GPU (0: skip the DI legs)")
    ap.add_argument("--no-quad", action="store_true", help="skip the 12D quadrotor leg (configs[3])")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def query_specs(rank: int, per_gpu: int, n: int):
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
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# --------------------------------------------------------------------------
def cpu_reference_leg(specs, lam: float, threads: int, reps: int):
    """The unmodified reference gmt_plan (oracle/_ref) over a sample of the
    same queries, one query per worker (simulator.cpp:212 pattern)."""
    import oracle
    R = oracle.ref()
    insts = R.instance_build_many(specs, threads)
    R.plan_many(insts, lam, threads)  # warm caches
    best = None
    secs = []
    for _ in range(reps):
        _, s = R.plan_many(insts, lam, threads)
        secs.append(s)
    sec = statistics.median(secs)
    best = len(insts) / sec
    # single-thread p50 of the first query (the CLI's plan_ms, gmtplan.cpp:144-152)
    t1 = []
    for _ in range(5):
        t0 = time.perf_counter()
        insts[0].plan(lam)
        t1.append(time.perf_counter() - t0)
    return best, statistics.median(t1) * 1e3, len(insts)


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    import oracle
    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libgmtref.so not built"}))
        return
    threads = os.cpu_count() or 1
    sample = min(args.cpu_sample, args.queries)
    specs = query_specs(0, sample, args.n)
    R = oracle.ref()
    insts = R.instance_build_many(specs, threads)
    for _ in range(args.warmup):
        R.plan_many(insts, 1.0, threads)
    secs = []
    for _ in range(args.steps):
        _, s = R.plan_many(insts, 1.0, threads)
        secs.append(s)
    total = sum(secs)
    value = len(insts) * args.steps / total
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": "forest3d_n4000_batched", "n": args.n, "dim": 3, "boxes": 60,
                   "lambda": 1.0, "queries_per_step": len(insts)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{len(insts)} queries of the workload per step, "
                                   f"gmt_plan(workers=1) per query under parallel_chunks({threads})"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
def run_b200(args):
    import numpy as np
    import torch

    from paper_1705_02403_b200 import abi, problem as P
    from paper_1705_02403_b200.shard import weak_range
    from paper_1705_02403_b200 import native
    from paper_1705_02403_b200.native import (OPT_BATCH_CLUSTER, OPT_BATCH_THREADS, OPT_COUNTERS,
                                              Context, PackedBatch, plan_batch_host)

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

    # ---- setup: build every query's instance on the GPU -------------------
    Q = args.queries
    specs = query_specs(rank, Q, args.n)
    insts = [ctx.build_instance(s) for s in specs]
    batch = ctx.batch(insts, 1.0)

    # instrumented launch (untimed): algorithmic traffic of one step
    ctx.set_option(OPT_COUNTERS, 1)
    ctx.counters(reset=True)
    cbatch = ctx.batch(insts, 1.0)
    cbatch.launch()
    cnt = ctx.counters(reset=True)
    ctx.set_option(OPT_COUNTERS, 0)
    sums = cbatch.summaries()
    cbatch.close()
    passes = sum(s.num_stats for s in sums)
    Vpasses = sum(s.num_stats * i.n for s, i in zip(sums, insts))
    b_alg = 12 * cnt["in_scan"] + 4 * cnt["out_scan"] + 8 * cnt["open_parent_reads"] + 9 * Vpasses
    ok = sum(1 for s in sums if s.status == abi.PLAN_SUCCESS)

    # ---- device-resident timed loop ---------------------------------------
    # A batched launch lasts as long as its slowest query; with --inflight S
    # the steps rotate over S contexts (streams, result buffers), so step k+1
    # fills the SMs that step k's finished queries left idle.  Every step is
    # still one complete 512-query batch; the timed region is bracketed by
    # events on the first stream, the others joined to it on both sides.
    S = max(1, args.inflight)
    lanes = [(ctx, stream, batch)]
    for _ in range(S - 1):
        c2 = Context(local)
        st2 = torch.cuda.ExternalStream(c2.stream, device=torch.device("cuda", local))
        lanes.append((c2, st2, c2.batch(insts, 1.0)))
    for _ in range(args.warmup):
        for _, _, b in lanes:
            b.launch()
    for c, _, _ in lanes:
        c.synchronize()
    barrier_sync()
    launches0 = sum(c.launch_count for c, _, _ in lanes)
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    joins = [torch.cuda.Event() for _ in lanes]
    with ClockSampler(local) as clk:
        start.record(stream)
        for _, st, _ in lanes[1:]:
            st.wait_event(start)
        for k in range(args.steps):
            lanes[k % S][2].launch()
        for (_, st, _), j in zip(lanes[1:], joins[1:]):
            j.record(st)
            stream.wait_event(j)
        end.record(stream)
        barrier_sync()
        for c, _, _ in lanes:
            c.synchronize()
    launches = sum(c.launch_count for c, _, _ in lanes) - launches0
    total_ms = max_over_ranks(start.elapsed_time(end))
    value = world * Q * args.steps / (total_ms / 1e3)
    kernel_ms = total_ms / args.steps  # effective time per solve launch (S in flight)
    # one launch alone (no overlap), for the record
    solo = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        batch.launch()
        e1.record(stream)
        e1.synchronize()
        solo.append(e0.elapsed_time(e1))
    solo_ms = statistics.median(solo)
    peak, peak_kind = measured_peak_hbm()
    achieved = b_alg / (kernel_ms / 1e3) / 1e9
    clocks = clk.summary()
    traffic, traffic_src = ncu_traffic("gmt_solve_kernel<1>:forest3d_n4000_q512")

    # ---- e2e through the C-ABI drop-in with host buffers ------------------
    entries = []
    for s, inst in zip(specs, insts):
        coords, gidx, g = inst.download()
        entries.append((s, coords, len(gidx), g, inst.init_index))
    pb = PackedBatch(entries, want_tree=True)
    for _ in range(max(1, args.warmup)):
        plan_batch_host(ctx, pb, 1.0)
    e2e_steps = max(3, min(args.steps, 20))
    barrier_sync()
    t = []
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        plan_batch_host(ctx, pb, 1.0)  # synchronous: returns with results on the host
        t.append(time.perf_counter() - t0)
    e2e_s = max_over_ranks(sum(t))
    e2e_graph_value = world * Q * e2e_steps / e2e_s
    # ---- e2e from problem descriptions: gmt_plan_problems (the step's scenes
    # in, summaries out; the offline phase -- sampling, init append, r-disk
    # graphs -- is inside the timed region, batched on the device) ----------
    from paper_1705_02403_b200.native import ProblemBatch
    pbatch = ProblemBatch(specs)  # the step's problem descriptions (host structs)
    for _ in range(max(1, args.warmup)):
        ctx.plan_problems(pbatch)
    barrier_sync()
    tp = []
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        pst, psum, _ = ctx.plan_problems(pbatch)
        tp.append(time.perf_counter() - t0)
    e2e_single_value = world * Q * e2e_steps / max_over_ranks(sum(tp))
    # two calls in flight: S host threads, one context (stream + scratch) each,
    # every thread planning the whole step's problems e2e_steps times; one
    # thread's offline build fills the SMs the other's solve tail leaves idle
    import threading
    pctx = [ctx] + [c for c, _, _ in lanes[1:S]]
    while len(pctx) < 2:
        pctx.append(Context(local))
    pctx = pctx[:2]
    thread_out = [None] * len(pctx)

    def _calls(i, k):
        for _ in range(k):
            thread_out[i] = pctx[i].plan_problems(pbatch)

    for c in pctx[1:]:
        c.plan_problems(pbatch)  # warm the second context's scratch
    barrier_sync()
    th = [threading.Thread(target=_calls, args=(i, e2e_steps)) for i in range(len(pctx))]
    t0 = time.perf_counter()
    for x in th:
        x.start()
    for x in th:
        x.join()
    e2e_mt_s = max_over_ranks(time.perf_counter() - t0)
    e2e_mt_value = world * Q * e2e_steps * len(pctx) / e2e_mt_s
    e2e_calls = len(pctx) if e2e_mt_value > e2e_single_value else 1
    e2e_value = max(e2e_mt_value, e2e_single_value)
    for i in range(len(pctx)):
        st_i, sum_i, _ = thread_out[i]
        if any(a != 0 for a in st_i) or [(a.status, a.cost, a.iterations) for a in sum_i] != \
                [(b.status, b.cost, b.iterations) for b in psum]:
            raise SystemExit("e2e results of the threaded calls differ from the single-thread ones")
    prob_h2d = sum(96 + 8 + 16 * s.dim * s.num_boxes + 24 * s.dim for s in specs)
    prob_d2h = Q * (40 + 16) + 8
    # parity spot check of the e2e results against the device-resident ones
    dev0 = batch.summaries()
    mism = sum(1 for a, b in zip(dev0, pb.summaries) if (a.status, a.cost, a.iterations) !=
               (b.status, b.cost, b.iterations))
    if mism:
        raise SystemExit(f"e2e results differ from device-resident results in {mism} queries")
    mism = sum(1 for a, st, b in zip(dev0, pst, psum) if st != 0 or (a.status, a.cost, a.iterations) !=
               (b.status, b.cost, b.iterations))
    if mism:
        raise SystemExit(f"problem-path results differ from device-resident results in {mism} queries")

    # ---- single-query latency (configs[1] canonical instance) -------------
    def single_p50(inst):
        out = {}
        for cs in (8, 16):
            ctx.set_option(OPT_BATCH_CLUSTER, cs)
            ctx.set_option(OPT_BATCH_THREADS, 0)
            b1 = ctx.batch([inst], 1.0)
            ctx.set_option(OPT_BATCH_CLUSTER, 0)
            for _ in range(5):
                b1.launch()
            ctx.synchronize()
            times = []
            with torch.cuda.stream(stream):
                for _ in range(args.single_reps):
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    b1.launch()
                    e1.record(stream)
                    e1.synchronize()
                    times.append(e0.elapsed_time(e1))
            out[f"cluster{cs}"] = statistics.median(times)
            b1.close()
        return out

    c2 = ctx.build_instance(P.forest_3d(3, args.n))
    single = single_p50(c2)
    p50 = min(single.values())

    # ---- configs[2] / configs[4]: the 6D double integrator -----------------
    di = None
    if args.di_queries > 0:
        t0 = time.perf_counter()
        c3 = ctx.build_instance(P.di_forest(3, args.n))
        ctx.synchronize()
        build_ms = (time.perf_counter() - t0) * 1e3
        s3 = single_p50(c3)
        di_insts = [ctx.build_instance(P.random_di_query(MASTER_SEED, q, n=args.n))
                    for q in weak_range(args.di_queries, rank)]
        bdis = [(c, st, c.batch(di_insts, 1.0)) for c, st, _ in lanes]  # same --inflight as the C2 leg
        bdi = bdis[0][2]
        for _ in range(args.warmup):
            for _, _, b in bdis:
                b.launch()
        for c, _, _ in bdis:
            c.synchronize()
        barrier_sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        di_launches = 6 * len(bdis)
        e0.record(stream)
        for _, st, _ in bdis[1:]:
            st.wait_event(e0)
        for k in range(di_launches):
            bdis[k % len(bdis)][2].launch()
        for _, st, _ in bdis[1:]:
            j = torch.cuda.Event()
            j.record(st)
            stream.wait_event(j)
        e1.record(stream)
        barrier_sync()
        for c, _, _ in bdis:
            c.synchronize()
        di_ms = max_over_ranks(e0.elapsed_time(e1) / di_launches)
        di = {"workload": "di6d_forest_n4000 (configs[2]) / batched random DI queries (configs[4])",
              "radius": c3.radius, "mean_out_degree": c3.num_edges / c3.n,
              "device_build_ms": build_ms, "p50_ms_single_solve": min(s3.values()),
              "single_solve_ms": s3, "batched_plans_per_s": world * len(di_insts) / (di_ms / 1e3),
              "batched_queries_per_gpu": len(di_insts), "batches_in_flight": len(bdis),
              "solved": sum(1 for s in bdi.summaries() if s.status == abi.PLAN_SUCCESS)}
        for _, _, b in bdis:
            b.close()

    # ---- configs[3]: the 12D linearised quadrotor, n = 8000 ---------------
    quad = None
    if not args.no_quad:
        spec4 = P.quad_scene()
        t0 = time.perf_counter()
        c4 = ctx.build_instance(spec4)
        ctx.synchronize()
        build_ms = (time.perf_counter() - t0) * 1e3
        s4 = single_p50(c4)
        r4 = ctx.plan(c4)
        quad = {"workload": "quad12d_scene_n8000 (configs[3]): 90 pillars + 40 beams",
                "radius": c4.radius, "weight": spec4.quad_weight, "n": c4.n,
                "mean_out_degree": c4.num_edges / c4.n, "goal_samples": c4.goal_count,
                "device_build_ms": build_ms, "p50_ms_single_solve": min(s4.values()),
                "single_solve_ms": s4, "status": r4.status, "cost": r4.cost,
                "iterations": r4.iterations, "collision_checks": r4.total_collision_checks}

    # ---- gather: one record per query to rank 0 (the only collective) -----
    from paper_1705_02403_b200.shard import gather_records, records
    recs = gather_records(records(dev0), device=f"cuda:{local}")

    line = None
    if rank == 0:
        cpu = None
        if not args.no_cpu:
            try:
                import oracle
                if oracle.ref_available():
                    threads = os.cpu_count() or 1
                    sample = min(args.cpu_sample, Q)
                    val, st_ms, nq = cpu_reference_leg(specs[:sample], 1.0, threads, 3)
                    cpu = {"value": val, "unit": UNIT, "cores": threads, "kind": "reference",
                           "sample": f"{nq} of the step's queries, median of 3 passes, "
                                     f"gmt_plan(workers=1) per query on {threads} threads; "
                                     f"single-thread p50 of query 0 = {st_ms:.2f} ms"}
            except Exception as e:  # the baseline must never break the bench line
                cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                       "sample": f"failed: {e}"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "forest3d_n4000_batched", "n": args.n, "dim": 3, "boxes": 60,
                       "lambda": 1.0, "queries_per_gpu_per_step": Q, "parallelism": f"dp{world}",
                       "batches_in_flight": S,
                       "l2": "inputs larger than L2 (per-GPU resident graphs ~%.1f GB)" %
                             (sum(i.num_edges for i in insts) * 12 / 1e9),
                       "solved": f"{int((recs[:, 0] == 0).sum())}/{len(recs)} success"},
            "p50_ms_single_solve": p50,
            "double_integrator_6d": di,
            "quadrotor_12d": quad,
            "single_solve_ms": single,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": prob_h2d,
                    "d2h_bytes_per_step": prob_d2h,
                    "path": "gmt_plan_problems: scenes in (host), summaries out; offline build + solve timed",
                    "calls_in_flight": e2e_calls,
                    "one_call_at_a_time": e2e_single_value,
                    "two_host_threads": e2e_mt_value},
            "e2e_host_graphs": {"value": e2e_graph_value, "unit": UNIT, "h2d_bytes_per_step": pb.h2d_bytes,
                                "d2h_bytes_per_step": pb.d2h_bytes,
                                "path": "gmt_plan_batch_host: host samples + CSR graphs in, summaries/paths/trees out"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_kind": peak_kind,
                         "kernel": "gmt_solve_kernel<1>",
                         "bytes_per_launch": b_alg, "kernel_ms": kernel_ms,
                         "kernel_ms_note": f"effective ms per launch with {S} launches in flight; one launch "
                                           f"alone takes {solo_ms:.3f} ms ({b_alg / solo_ms / 1e6:.0f} GB/s)",
                         "counts": {**cnt, "passes": passes, "V_passes": Vpasses}},
            "cpu_baseline": cpu,
            "clocks": clocks,
            "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return line


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
