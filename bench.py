#!/usr/bin/env python
"""Benchmark of the B200 sliced contraction-tree executor.

    python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference]

One "step" = one slice of BASELINE.json configs[3] (rectangular 7x7 (1+40+1)
random-circuit amplitude, 742 rank-3 tensors, reference min-fill tree, sliced
by greedy_slice to W_s = 27) per GPU.  The timed slices are drawn from the
workload's list of slices that are nonzero in exact arithmetic
(benchdata/cfg4_7x7_d40.slices.json, found by tools/slice_scan.py); every rank
contracts its own block of that list (weak scaling, no data-path collective)
and the per-rank complex128 partial sums meet in one NCCL all-reduce.

Metric: effective contraction FLOP/s = 8 * C_s(executed) / t,
reported in TFLOP/s, whole job over all ranks, with slices/s alongside.
Inputs are resident in HBM for `value`; `e2e` re-binds the leaves from pinned
host memory and reads the result back every step through the public API.
Also in the line: the roofline against the measured tensor-pipe ceiling at the
measured SM clock, a >= 10 s sustained run, the CPU oracle on one slice with
the slice's parity, and a short run of configs[4] (`secondary`).  The
per-slice working set (11 GB of intermediates) exceeds the 126 MB L2, so no
explicit L2 flush is needed between timed slices.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

WORKLOAD = "cfg4_7x7_d40"
METRIC = "effective contraction FLOP/s (8*C_s/t), sliced 7x7 (1+40+1) circuit amplitude"

_REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
            0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
            0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
            0x100: "display_clock_setting"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,power.draw",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return self

        def reader():
            for line in self.proc.stdout:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 4:
                    try:
                        self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16),
                                             float(parts[3])))
                    except ValueError:
                        pass

        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()
        time.sleep(0.25)
        return self

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        self.proc.wait(timeout=5)
        self.thread.join(timeout=2)
        busy = [s for s in self.samples if not (s[2] & 0x1)] or self.samples
        if not busy:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        mhz = sorted(s[0] for s in busy)
        reasons = set()
        for s in busy:
            for bit, name in _REASONS.items():
                if s[2] & bit and bit != 0x1:
                    reasons.add(name)
        return {"sm_mhz": mhz[len(mhz) // 2], "sm_max_mhz": max(s[1] for s in busy),
                "reasons": sorted(reasons), "samples": len(busy),
                "power_w_max": max(s[3] for s in busy)}


def load_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            p = json.load(fh)
        return p, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def load_traffic():
    """DRAM traffic of the dominant tensor-core launch of a bench slice, from
    the committed ncu launch list with dram metrics (tools/summarize_profiles.py
    inslice_traffic); falls back to the standalone full capture."""
    path = os.path.join(REPO, "profiles", "r02_gemm_inslice_traffic.json")
    if os.path.exists(path):
        with open(path) as fh:
            t = json.load(fh)
        d = t["dominant"]
        return {"dram_bytes_per_launch": d["dram_bytes"], "algorithmic_bytes": d["algorithmic_bytes"],
                "kernel": (f"gemm_c64_3xtf32 in-slice v{d['ssa']} M={d['M']} N={d['N']} K={d['K']} "
                           f"(profiles/r02_gemm_inslice_traffic.json: {d['ratio']:.2f}x its algorithmic bytes; "
                           f"all tensor-core launches of the slice {t['all_gemm_ratio']:.2f}x)")}
    path = os.path.join(REPO, "profiles", "ncu_gemm_traffic.json")
    if os.path.exists(path):
        with open(path) as fh:
            return json.load(fh)
    return None


def load_mma_peak():
    """Committed MMA-only ceiling (tools/mma_peak.py output), if present."""
    for name in ("r02_mma_peak.json",):
        path = os.path.join(REPO, "profiles", name)
        if os.path.exists(path):
            with open(path) as fh:
                return json.load(fh), f"profiles/{name}"
    return None, None


def workload(args):
    from paper_2002_01935_b200.harness.workloads import load_workload
    if args.ws == "auto":
        import torch
        from paper_2002_01935_b200.slicing import auto_slice
        tn, tree, _, meta = load_workload(args.config, ws=1e9)
        free, _total = torch.cuda.mem_get_info()
        ss, need = auto_slice(tree, tn, free, ws_max=40)
        meta["ws_auto"] = {"device_free_bytes": free, "plan_bytes": need}
        return tn, tree, ss, meta
    return load_workload(args.config, ws=None if args.ws is None else float(args.ws))


def cpu_baseline(tn, tree, ss, slice_id, budget_s):
    """Oracle (port of the reference per-op semantics, complex128, OpenBLAS on
    every host core) on one slice of the same workload."""
    import numpy as np
    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover
        threadpool_limits = None
    import oracle
    from paper_2002_01935_b200.slicing import slice_assignment
    cores = len(os.sched_getaffinity(0))
    asg = slice_assignment(tn, ss, slice_id)
    ctx = threadpool_limits(limits=cores) if threadpool_limits else None
    rec = {}
    root = tree.root
    keep = {root}
    if tree.n > 1:
        keep.update(tree.children(root))

    class _Rec(dict):  # keep only the root and its operands
        def __setitem__(self, k, v):
            if k in keep:
                dict.__setitem__(self, k, v)

    rec = _Rec()
    t0 = time.perf_counter()
    try:
        r, _, ops, _ = oracle.contract_one(tn, tree, ss.labels, asg, record=rec)
    finally:
        if ctx is not None:
            ctx.__exit__(None, None, None)
    dt = time.perf_counter() - t0
    scale = None
    if tree.n > 1:
        a, b = tree.children(root)
        scale = float(np.linalg.norm(rec[a][1].ravel()) * np.linalg.norm(rec[b][1].ravel())) if (
            a in rec and b in rec) else None
    return complex(np.asarray(r)), ops, dt, cores, scale


def run_reference(args):
    """--impl reference: the reference's CPU path (oracle port; the reference
    ships no executor) on the host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    tn, tree, ss, meta = workload(args)
    from paper_2002_01935_b200.refpkg import annotate_incidence
    annotate_incidence(tree, tn)
    import oracle
    per_slice = oracle.width_cost(tn, tree, ss.labels)[1]
    flops = 8 * per_slice
    times = []
    cores = len(os.sched_getaffinity(0))
    # each step is one slice; the number of timed steps is bounded so the run
    # stays within a few minutes of host time
    steps = args.steps
    warm = min(args.warmup, 1)
    budget = args.ref_budget
    spent = 0.0
    nz_path = os.path.join(REPO, "benchdata", f"{args.config}.slices.json")
    ids = [i % int(ss.d) for i in range(warm + steps)]  # unsliced / few-slice configs repeat
    if args.slices == "nonzero" and os.path.exists(nz_path):
        with open(nz_path) as fh:
            nz_rec = json.load(fh)
        if float(nz_rec["ws"]) == float(ss.Ws) and str(nz_rec.get("d", ss.d)) == str(ss.d):
            ids = [int(x) for x in nz_rec["ids"]][:warm + steps]  # the b200 arm's rank-0 ids
    for i in range(len(ids)):
        val, ops, dt, cores, _ = cpu_baseline(tn, tree, ss, ids[i], budget)
        assert ops == per_slice
        spent += dt
        if i >= warm:
            times.append(dt)
        if spent > budget and len(times) >= 1:
            break
    t = sum(times)
    value = len(times) * flops / t / 1e12
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s",
            "n_gpus": args.gpus, "steps": len(times), "warmup": warm,
            "ms_per_step": 1e3 * t / len(times), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": args.config, "W_s": ss.Ws, "slices_total": str(ss.d),
                       "flops_per_slice": flops},
            "slices_per_s": len(times) / t,
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "port",
                             "sample": f"{len(times)} full slice(s) of {args.config} (W_s={ss.Ws:g}; ids "
                                       f"{ids[warm:warm + len(times)]}), "
                                       "oracle restatement of SPEC contract_sliced over the reference's "
                                       "pairwise_contract/fix_index semantics, complex128 numpy einsum"},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def measure_secondary(name, torch, stream, probe, sms, W=2, K=8):
    """A short timed run of another BASELINE workload (its default W_s, slice
    prefix or all slices), reported beside the headline: TFLOP/s, mean SM
    clock (cycle stamps) and the fraction of the split-TF32 ceiling at it."""
    from paper_2002_01935_b200 import _native
    from paper_2002_01935_b200.executor import SlicedPlan
    from paper_2002_01935_b200.harness.workloads import load_workload
    tn, tree, ss, meta = load_workload(name)
    plan = SlicedPlan(tn, tree, ss).bind()
    try:
        ids = [i % plan.d for i in range(W + K)]
        for s_ in ids[:W]:
            plan.run(s_, s_ + 1, stream)
        torch.cuda.synchronize()
        stamps = _native.ClockStamps()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stamps.start(stream.cuda_stream)
        e0.record(stream)
        for s_ in ids[W:]:
            plan.run(s_, s_ + 1, stream)
        e1.record(stream)
        stamps.stop(stream.cuda_stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        mhz, _ = stamps.mhz()
        flops = plan.flops_per_slice
        value = K * flops / (ms / 1e3) / 1e12
        peak = probe["tf32_flop_per_clk_per_sm"] * sms * mhz * 1e6 / 1e12 / 3.0 if probe and mhz else None
        return {"workload": name, "desc": meta["desc"], "W": meta["W"], "log10_C": meta["log10_C"],
                "W_s": ss.Ws, "d_sliced": str(ss.d), "flops_per_slice": flops, "steps": K,
                "value": value, "unit": "TFLOP/s", "ms_per_step": ms / K, "slices_per_s": K / (ms / 1e3),
                "sm_mhz_cycles": mhz, "roofline_peak": peak, "frac": value / peak if peak else None,
                "tree_source": meta["tree_source"]}
    finally:
        plan.close()


def spawn_ranks(n):
    """`bench.py --gpus N` without a launcher: start one rank per GPU under
    torch.distributed.run (127.0.0.1 rendezvous) and return its exit code.
    Each child sees WORLD_SIZE and runs the per-rank path below."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


NOMINAL_TF32 = 1100.0  # TFLOP/s dense, B200 (context only)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=WORKLOAD)
    ap.add_argument("--ws", default=None, help="target sliced width, or 'auto' (largest W_s whose plan fits HBM)")
    ap.add_argument("--precision", default="3xtf32", choices=["3xtf32", "tf32-bf16x", "fp32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=90.0)
    ap.add_argument("--profile-out", default=None)
    ap.add_argument("--no-tf32-probe", action="store_true", help="skip the live MMA-only ceiling probe")
    ap.add_argument("--slices", default="nonzero", choices=["nonzero", "prefix"],
                    help="timed slice ids: the workload's nonzero-slice list (benchdata/<config>.slices.json) "
                         "or the enumeration prefix")
    ap.add_argument("--secondary", default="cfg5_syc53_m12",
                    help="comma-separated workloads timed briefly after the headline ('' to skip)")
    ap.add_argument("--sustained-s", type=float, default=10.0,
                    help="after the headline, time ~this many seconds of further slices (0: skip)")
    ap.add_argument("--no-direct", action="store_true", help="disable GEMM->GEMM operand-plane fusion")
    ap.add_argument("--force-dist", action="store_true",
                    help="initialise torch.distributed even at world size 1 (exercises the NCCL path)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)

    import numpy as np
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; reporting the {world} ranks that run",
              file=sys.stderr)
    # TNX_BENCH_BACKEND=gloo lets the multi-rank logic be exercised with
    # several ranks sharing one GPU (no kernel waits on another rank); the
    # production path is NCCL with one GPU per rank.
    backend = os.environ.get("TNX_BENCH_BACKEND", "nccl")
    local = local % torch.cuda.device_count() if backend != "nccl" else local
    torch.cuda.set_device(local)
    use_dist = world > 1 or args.force_dist
    if use_dist:
        if "MASTER_ADDR" not in os.environ:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    from paper_2002_01935_b200.executor import SlicedPlan
    from paper_2002_01935_b200.distributed import slice_range, allreduce_complex
    t_setup = time.perf_counter()
    tn, tree, ss, meta = workload(args)
    plan = SlicedPlan(tn, tree, ss, device=local, precision=args.precision,
                      direct_planes=not args.no_direct)
    plan.bind()
    setup_s = time.perf_counter() - t_setup
    st = plan.stats()
    flops_slice = plan.flops_per_slice
    W, K = args.warmup, args.steps
    nz_path = os.path.join(REPO, "benchdata", f"{args.config}.slices.json")
    use_list = args.slices == "nonzero" and os.path.exists(nz_path)
    if use_list:
        with open(nz_path) as fh:
            nz_rec = json.load(fh)
        nz_ids = [int(x) for x in nz_rec["ids"]]
        # the list belongs to one slice set (the workload's default W_s)
        use_list = float(nz_rec["ws"]) == float(ss.Ws) and str(nz_rec.get("d", ss.d)) == str(ss.d)
    cyc = (not use_list) and (W + K) * world > plan.d  # few slices (or unsliced): repeat them
    # an explicit stream: the legacy default stream has handle 0, which the C
    # ABI reads as "the library's own stream"
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    # Which slices the job contracts.  "nonzero" (default when the workload has
    # a benchdata/<config>.slices.json list): ids that are nonzero in exact
    # arithmetic, found by tools/slice_scan.py -- the timed operands are then
    # real amplitude data, not round-off of structurally zero slices (which
    # draw less power); rank r takes the r-th block of W+K ids, cycling
    # through the list.  "prefix": the prefix [0, world*(W+K)) of the slice
    # enumeration, one contiguous block per rank (bit-exact sub-range).
    base = slice_range(0, world * (W + K), world, rank)[0] if not cyc else rank * (W + K)

    def job_ids(offset, n):
        if use_list:
            return [nz_ids[(offset + i) % len(nz_ids)] for i in range(n)]
        if cyc:
            return [(offset + i) % plan.d for i in range(n)]
        return list(range(offset, offset + n))

    warm_ids = job_ids(rank * (W + K) if use_list else base, W)
    timed_ids = job_ids(rank * (W + K) + W if use_list else base + W, K)

    def run_ids(ids):
        """Contract `ids` into the accumulator in one library call
        (tnx_run_slice_ids: consecutive runs replay the graph back to back)."""
        plan.run_ids(ids, stream)
    red_dev = "cuda" if backend == "nccl" else "cpu"

    def barrier():
        if use_dist:
            if backend == "nccl":
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()

    # warm-up
    run_ids(warm_ids)
    torch.cuda.synchronize()
    plan.reset(stream)
    torch.cuda.synchronize()

    # timed region: K slices per rank, graph replays on the torch stream
    clk = ClockSampler(local).start()
    barrier()
    torch.cuda.synchronize()
    from paper_2002_01935_b200 import _native
    stamps = _native.ClockStamps()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    stamps.start(stream.cuda_stream)
    e0.record(stream)
    run_ids(timed_ids)
    e1.record(stream)
    stamps.stop(stream.cuda_stream)
    torch.cuda.synchronize()
    barrier()
    clocks = clk.stop()
    # mean SM clock over the timed slices from the SMs' own cycle counters
    # (clock64 / globaltimer stamps on the stream before and after)
    clocks["sm_mhz_cycles"], clocks["sm_cycle_stamps"] = stamps.mhz()
    ms = e0.elapsed_time(e1)
    t_max = torch.tensor([ms], dtype=torch.float64, device=red_dev)
    if use_dist:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms_max = float(t_max.item())

    def slice_values(ids):
        """Per-slice values of `ids` (each contracted alone, not accumulated)."""
        vals = []
        for s_ in ids:
            plan.reset(stream)
            plan.run(s_, s_ + 1, stream)
            vals.append(complex(np.asarray(plan.result(stream)).ravel()[0]))
        return vals

    def zero_fraction(vals):
        """Slices whose value is zero in exact arithmetic: |v| below 1e-8 of the
        largest |v| of the sample (they come out at ~1e-16 of it, noise)."""
        big = max((abs(v) for v in vals), default=0.0)
        return sum(1 for v in vals if abs(v) <= 1e-8 * big) / len(vals) if vals and big > 0 else None

    # final exchange: one all-reduce of the complex128 partial sums
    part = plan.result(stream)
    a0 = time.perf_counter()
    total = allreduce_complex(part, device=red_dev)
    torch.cuda.synchronize()
    allreduce_ms = 1e3 * (time.perf_counter() - a0)

    total_slices = K * world
    value = total_slices * flops_slice / (ms_max / 1e3) / 1e12
    slices_per_s = total_slices / (ms_max / 1e3)
    timed_zero = zero_fraction(slice_values(timed_ids)) if st["out_elements"] == 1 else None

    # per-launch profile of one slice (CUDA events on the launching stream)
    # (the profile runs right after the headline, before the sustained run heats
    # the GPU; its own mean SM clock prices the per-kernel roofline)
    torch.cuda.synchronize()
    stamps.start(stream.cuda_stream)
    torch.cuda.synchronize()
    prof_b = plan.profile_slice(timed_ids[0], with_bytes=True)
    torch.cuda.synchronize()
    stamps.stop(stream.cuda_stream)
    torch.cuda.synchronize()
    prof_mhz, _ = stamps.mhz()
    prof = [(k, v, t) for k, v, t, b in prof_b]
    info = {v["ssa"]: v for v in plan.vertex_info()}
    gemm_ms = sum(t for k, v, t in prof if k == "gemm")
    gemm_flops = sum(8 * info[v]["macs"] for k, v, t in prof if k == "gemm")
    n_gemm = sum(1 for k, v, t in prof if k == "gemm")
    slice_ms = sum(t for _, _, t in prof)
    peaks, peak_kind = load_peaks()
    # Roofline denominator: the tensor pipe's own ceiling, measured live by an
    # MMA-only tcgen05.mma kind::tf32 loop (tnx_mma_peak: no TMA, no epilogue,
    # operands resident in shared memory, one CTA pair per SM pair), divided
    # by 3 (split-TF32: 24 M N K real tensor flop per 8 M N K complex flop).
    probe = None
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    if not args.no_tf32_probe:
        best = None
        for cg in (2, 1):
            _native.mma_peak("tf32", cg, 20000, stream.cuda_stream)
            t, mhz, pms = _native.mma_peak("tf32", cg, 150000, stream.cuda_stream)
            if best is None or t / mhz > best[0] / best[1]:
                best = (t, mhz, pms, cg)
        probe = {"tf32_tflops": best[0], "sm_mhz": best[1], "ms": best[2], "cta_group": best[3],
                 "tf32_flop_per_clk_per_sm": best[0] * 1e12 / (best[1] * 1e6) / sms}
        _native.mma_peak("ffma", 1, 20000, stream.cuda_stream)
        f_t, f_mhz, _ = _native.mma_peak("ffma", 1, 200000, stream.cuda_stream)
        probe.update({"ffma_tflops": f_t, "ffma_sm_mhz": f_mhz,
                      "ffma_flop_per_clk_per_sm": f_t * 1e12 / (f_mhz * 1e6) / sms})
    committed, committed_src = load_mma_peak()
    timed_mhz = clocks.get("sm_mhz_cycles") or clocks.get("sm_mhz")
    prof_clock = prof_mhz or timed_mhz
    if probe and prof_clock:
        # the probe's per-clock rate at the clock the timed slices ran at (the
        # MMA-only loop on random operands draws more power than the GEMM and
        # runs at a lower clock, so its raw TFLOP/s would understate the ceiling)
        p_c = probe["tf32_flop_per_clk_per_sm"] * sms * prof_clock * 1e6 / 1e12 / 3.0
        peak_src = (f"live tnx_mma_peak (tcgen05.mma kind::tf32 MMA-only loop, cta_group::{probe['cta_group']}): "
                    f"{probe['tf32_flop_per_clk_per_sm']:.0f} flop/clk/SM x {sms} SMs x {prof_clock:.0f} MHz "
                    f"(mean SM clock over the per-launch profile the achieved figure comes from, "
                    f"clock64/globaltimer stamps) / 3 split-TF32 passes; raw probe {probe['tf32_tflops']:.1f} TFLOP/s at {probe['sm_mhz']:.0f} MHz")
    elif probe:
        p_c = probe["tf32_tflops"] / 3.0
        peak_src = (f"live tnx_mma_peak: tcgen05.mma kind::tf32 MMA-only loop, cta_group::{probe['cta_group']}, "
                    f"{probe['tf32_tflops']:.1f} TFLOP/s at {probe['sm_mhz']:.0f} MHz (CTA clock64/globaltimer) "
                    f"/ 3 split-TF32 passes")
    elif committed:
        p_c = committed["complex_3xtf32_peak_tflops"]
        peak_src = f"{committed_src}: MMA-only kind::tf32 {committed['tf32_peak_tflops']:.1f} TFLOP/s / 3"
    else:
        p_c = peaks["bf16_tflops"] / 2.0 / 3.0
        peak_src = (f"{peak_kind} MEASURED_PEAKS bf16_tflops {peaks['bf16_tflops']} / 2 (TF32 = half the "
                    f"BF16 tensor rate) / 3 (split-TF32 passes)")
    achieved = gemm_flops / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else 0.0
    traffic = load_traffic()
    # per-vertex roofline of the dominant contractions (top vertices covering
    # >= 90 % of the slice's FLOPs; the north-star criterion)
    per_v = {}
    for k, v, t in prof:
        if v >= 0:
            per_v.setdefault(v, {"gemm": 0.0, "other": 0.0})
            per_v[v]["gemm" if k == "gemm" else "other"] += t
    fl_total = 8 * sum(x["macs"] for x in info.values())
    dom, acc_fl = [], 0
    for v in sorted(info, key=lambda u: -info[u]["macs"]):
        if acc_fl >= 0.9 * fl_total or v not in per_v:
            break
        x = info[v]
        fl = 8 * x["macs"]
        t = per_v[v]["gemm"] + per_v[v]["other"]
        dom.append({"ssa": v, "kind": x["kind"], "M": x["m"], "N": x["n"], "K": x["k"], "ms": round(t, 4),
                    "flop_share": round(fl / fl_total, 4), "tflops": round(fl / t / 1e9, 1),
                    "frac": round(fl / t / 1e9 / p_c, 3)})
        acc_fl += fl
    # HBM roofline of the memory-bound kernels (permute / pack / dot): algorithmic
    # bytes per launch reported by the library
    mem_ms = sum(t for k, v, t, b in prof_b if k == "pack" or (k == "simt" and b > 0))
    mem_bytes = sum(b for k, v, t, b in prof_b if k == "pack" or (k == "simt" and b > 0))
    hbm = {"kernels": "perm_vec/perm/pack/dot", "achieved_gbs": mem_bytes / (mem_ms / 1e3) / 1e9 if mem_ms else None,
           "peak_gbs": peaks["hbm_gbs"], "frac": (mem_bytes / (mem_ms / 1e3) / 1e9 / peaks["hbm_gbs"]) if mem_ms else None,
           "ms_per_slice": mem_ms}
    # the aggregate is dominated by many sub-MB launches (latency-bound); the large
    # launches show the kernels' bandwidth
    big = [(t, b) for k, v, t, b in prof_b if (k == "pack" or (k == "simt" and b > 0)) and b >= 16e6]
    if big:
        bt, bb = sum(t for t, _ in big), sum(b for _, b in big)
        hbm["large_launches"] = {"min_bytes": 16e6, "count": len(big), "achieved_gbs": bb / (bt / 1e3) / 1e9,
                                 "frac": bb / (bt / 1e3) / 1e9 / peaks["hbm_gbs"]}
    small = [b for k, v, t, b in prof_b if (k == "pack" or (k == "simt" and b > 0)) and b < 16e6]
    hbm["small_launches"] = {"count": len(small), "median_bytes": float(np.median(small)) if small else None}
    # slice roofline: t*_v = max(8 U_v / P, 8 B x (|A|+|B|+|O|) / BW) per
    # per-slice vertex -- P = the split-TF32 ceiling for tensor-core vertices, the
    # FFMA ceiling (same clock) for SIMT ones -- summed and divided by the
    # measured slice time
    p_simt = (probe["ffma_flop_per_clk_per_sm"] * sms * prof_clock * 1e6 / 1e12
              if probe and prof_clock else None)
    t_star = 0.0
    if p_simt:
        bw = peaks["hbm_gbs"] * 1e9
        for x in info.values():
            if x["hoisted"]:
                continue
            byts = 8.0 * x["batch"] * (x["m"] * x["k"] + x["n"] * x["k"] + x["m"] * x["n"])
            pk = p_c if x["kind"] == "gemm_tc" else p_simt
            t_star += max(8.0 * x["macs"] / (pk * 1e12), byts / bw)
    slice_roofline = {"t_star_ms": 1e3 * t_star, "slice_ms": slice_ms,
                      "frac": 1e3 * t_star / slice_ms if slice_ms and t_star else None,
                      "p_simt_tflops": p_simt,
                      "def": "sum over per-slice vertices of max(8 U_v / P, 8 B (|A|+|B|+|O|) / HBM BW) "
                             "/ profiled slice time (P: split-TF32 ceiling for tensor-core vertices, "
                             "FFMA ceiling for SIMT vertices, both at the timed clock)"}
    by_kind = {}
    for k, v, t in prof:
        by_kind[k] = by_kind.get(k, 0.0) + t
    roofline = {"bound": "tensor", "achieved": achieved, "peak": p_c, "unit": "TFLOP/s",
                "frac": achieved / p_c if p_c else None,
                "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
                "traffic_note": (traffic.get("kernel") + "; algorithmic bytes " +
                                 str(traffic.get("algorithmic_bytes"))) if traffic else None,
                "kernel": "gemm_c64_3xtf32 (tcgen05.mma.kind::tf32, 4M x 3 split passes)",
                "peak_source": peak_src,
                "mma_probe": probe,
                "probe_peak_raw": probe["tf32_tflops"] / 3.0 if probe else None,
                "profile_sm_mhz_cycles": prof_mhz,
                # the whole timed slice (every kernel, launch gaps) against the same ceiling
                # at the timed region's own clock
                "value_frac_at_timed_clock": (value / (probe["tf32_flop_per_clk_per_sm"] * sms * timed_mhz
                                                       * 1e6 / 1e12 / 3.0) if probe and timed_mhz else None),
                "measured_peaks_bf16_context": peaks["bf16_tflops"] / 2.0 / 3.0,
                "gemm_share_of_slice": gemm_ms / slice_ms if slice_ms else None,
                "gemm_launches_per_slice": n_gemm,
                "time_share_ms": {k: round(t, 3) for k, t in by_kind.items()},
                "dominant_vertices": dom,
                "dominant_min_frac": min((d["frac"] for d in dom), default=None),
                # context: NVIDIA's nominal dense TF32 (1.1 PFLOP/s, B200_PROFILING.md) / 3 passes
                "nominal_peak": NOMINAL_TF32 / 3.0,
                "frac_nominal": achieved / (NOMINAL_TF32 / 3.0),
                "dominant_min_frac_nominal": min((d["tflops"] / (NOMINAL_TF32 / 3.0) for d in dom), default=None),
                "hbm_bound_kernels": hbm,
                "slice_roofline": slice_roofline}
    if args.profile_out and rank == 0:
        with open(args.profile_out, "w") as fh:
            json.dump({"launches": prof, "vertices": list(info.values())}, fh, default=str)

    # end-to-end through the public API: pinned host leaves -> bind -> slice -> D2H
    e2e = None
    if not args.no_e2e:
        leaves = []
        for nid in tree.leaves:
            a = torch.from_numpy(np.ascontiguousarray(tn.node(nid).data, dtype=np.complex128)).pin_memory()
            leaves.append(a.numpy())
        h2d = sum(a.nbytes for a in leaves)
        nout = max(1, st["out_elements"])
        d2h = 16 * nout
        res = torch.zeros((len(timed_ids), 2 * nout), dtype=torch.float64).pin_memory()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        # every step: H2D of the leaves (bind), the slice, and an async D2H of the
        # step's result into pinned host memory; one synchronisation at the end
        for i, sid_ in enumerate(timed_ids):
            plan.bind(leaf_arrays=leaves, stream=stream)
            plan.run(sid_, sid_ + 1, stream)
            plan.result_async(res[i], stream)
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        if not bool(torch.isfinite(res).all()):
            raise SystemExit("e2e: non-finite step result")
        t_e = torch.tensor([e2e_s], dtype=torch.float64, device=red_dev)
        if use_dist:
            dist.all_reduce(t_e, op=dist.ReduceOp.MAX)
        e2e_s = float(t_e.item())
        e2e = {"value": total_slices * flops_slice / e2e_s / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "slices_per_s": total_slices / e2e_s,
               "note": "each step: tnx_bind_leaves (H2D from pinned host + slice-invariant subtrees) + 1 slice "
                       "+ async D2H of the step's result into pinned host memory; one sync at the end"}

    # sustained: the same per-slice work for >= --sustained-s seconds (the GEMMs
    # run into the 1 kW power cap; the headline above is a ~0.5 s burst)
    sustained = None
    if args.sustained_s > 0:
        n_s = max(K, int(math.ceil(args.sustained_s * 1e3 / (ms_max / K))))
        s_base = world * (W + K) + rank * n_s
        sus_ids = job_ids(s_base, n_s)
        if use_list or cyc or s_base + n_s <= plan.d:
            plan.reset(stream)
            clk2 = ClockSampler(local).start()
            barrier()
            torch.cuda.synchronize()
            f0 = torch.cuda.Event(enable_timing=True)
            f1 = torch.cuda.Event(enable_timing=True)
            stamps.start(stream.cuda_stream)
            f0.record(stream)
            run_ids(sus_ids)
            f1.record(stream)
            stamps.stop(stream.cuda_stream)
            torch.cuda.synchronize()
            barrier()
            clocks2 = clk2.stop()
            clocks2["sm_mhz_cycles"], clocks2["sm_cycle_stamps"] = stamps.mhz()
            ms2 = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=red_dev)
            if use_dist:
                dist.all_reduce(ms2, op=dist.ReduceOp.MAX)
            ms2 = float(ms2.item())
            # a contiguous block (zero slices follow the sliced labels' digit
            # pattern, so a strided sample can alias with it)
            mid = max(0, n_s // 2 - 24)
            sample = sus_ids[mid:mid + 48]
            sustained = {"value": n_s * world * flops_slice / (ms2 / 1e3) / 1e12, "unit": "TFLOP/s",
                         "seconds": ms2 / 1e3, "slices_per_rank": n_s, "ms_per_step": ms2 / n_s,
                         "slices_per_s": n_s * world / (ms2 / 1e3), "clocks": clocks2,
                         "zero_slice_fraction": zero_fraction(slice_values(sample))
                         if st["out_elements"] == 1 else None,
                         "zero_sample": f"{len(sample)} consecutive slices from the middle of the sustained range"}

    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sid = timed_ids[0]
        plan.reset(stream)
        plan.run(sid, sid + 1, stream)
        gpu_val = complex(plan.result(stream))
        ref_val, ops, dt, cores, scale = cpu_baseline(tn, tree, ss, sid, 60)
        cpu = {"value": flops_slice / dt / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": "port",
               "sample": f"slice {sid} of {args.config} (one full slice, {flops_slice:.3e} flop), "
                         "oracle/ restatement in complex128 numpy (einsum -> OpenBLAS)",
               "seconds": dt, "slices_per_s": 1.0 / dt}
        parity = {"slice": sid, "gpu": [gpu_val.real, gpu_val.imag], "cpu": [ref_val.real, ref_val.imag],
                  "normwise_err": abs(gpu_val - ref_val) / scale if scale else None,
                  "normwise_def": "|c_gpu - c_cpu| / (||x_root|| ||y_root||), operands of the root "
                                  "contraction from the complex128 oracle",
                  "rel_err": abs(gpu_val - ref_val) / abs(ref_val) if ref_val != 0 else None}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": K,
                "warmup": W, "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": {"3xtf32": "c64 (3xTF32 tcgen05 + FP32 SIMT)",
                                               "tf32-bf16x": "c64 (TF32 hi*hi + BF16 cross terms, tcgen05)",
                                               "fp32": "c64 (FP32 SIMT)"}[args.precision],
                "data": "synthetic (seeded GRCS-style circuit, reference-driver tree)",
                "config": {"workload": args.config, "desc": meta["desc"], "W": meta["W"],
                           "log10_C": meta["log10_C"], "W_s": ss.Ws, "log10_Cs": ss.log10_Cs,
                           "d_sliced": str(ss.d), "sliced_labels": len(ss.labels),
                           "flops_per_slice": flops_slice, "slices_per_rank": K,
                           "l2": "per-slice working set > L2 (no flush needed)",
                           "slices": (f"nonzero slice ids ({len(nz_ids)} in benchdata/{args.config}.slices.json, "
                                      f"nonzero fraction of a random sample {nz_rec['nonzero_fraction']:.3f}); "
                                      f"rank r times ids [r*(W+K)+W, (r+1)*(W+K)) of the list, cyclic"
                                      if use_list else (f"slice ids cycling through all {plan.d} slices"
                                                        if cyc else
                                                        f"prefix [0, {world * (W + K)}) of the enumeration")),
                           "tree_source": meta["tree_source"], "precision": args.precision,
                           "ws_auto": meta.get("ws_auto")},
                "slices_per_s": slices_per_s,
                "zero_slice_fraction": timed_zero,
                "sustained": sustained,
                "roofline": roofline, "cpu_baseline": cpu, "parity": parity,
                "e2e": e2e, "clocks": clocks,
                "gpu_launches": K * st["launches_per_slice"],
                "plan": {k: st[k] for k in ("num_gemm", "num_simt", "num_hoisted", "launches_per_slice",
                                            "work_arena_bytes")},
                # context only (vs_baseline stays null: BASELINE.json lists no published number):
                # paper Table II, 7x7 (1+40+1), single precision on a Quadro P2000, Hyper-Par trees
                "paper_context": ({"effective_tflops": 1.353, "hardware": "NVIDIA Quadro P2000 (3.03 TFLOP/s FP32)",
                                   "source": "BASELINE.md §1 (PAPER.md:724-725, derived 8*C_s/t)",
                                   "ratio": value / 1.353} if args.config == WORKLOAD else None),
                "allreduce_ms": allreduce_ms, "setup_s": setup_s, "backend": backend if use_dist else None,
                "prefix_sum": [complex(np.asarray(total).ravel()[0]).real, complex(np.asarray(total).ravel()[0]).imag]}
    plan.close()
    if rank == 0:
        if world == 1 and args.config == WORKLOAD and args.secondary:
            line["secondary"] = [measure_secondary(name, torch, stream, probe, sms) for name in args.secondary.split(",")]
        print(json.dumps(line, default=str))
    if use_dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
