#!/usr/bin/env python3
"""Benchmark of the gear-plan sweep (headline) and the stage step.

Headline workload (BASELINE.json configs[1]): Sentiment-140-shaped 4-stage
cascade (BERT tiny/mini/small/base stand-ins m0..m3, cost ratios 1:4:16:64),
1M synthetic validation samples with the reference make_validation
semantics, 100-level threshold grids per model -> the full cascade x
threshold product, C = 1,040,604 configs.  One step = one full sweep
(histogram + prefix tables + every config's accuracy / mean_cost /
forward_frac) with inputs resident in HBM.  Metric: config-evals/s.

`e2e`: the same sweep through the public API from HOST buffers: pinned
H2D of the certainty / correct matrices, sweep, exact Pareto front, D2H of
the front (config index, accuracy, mean_cost, forward_frac) every step.

Multi-GPU (torchrun): weak scaling — every rank sweeps its own tenant's
validation set (per-GPU work fixed) and the ranks all-gather their Pareto
fronts over NCCL each step (distributed.gather_fronts).

--impl reference: the reference algorithm's CPU implementation (the oracle
port of _evaluate_numba, oracle/oracle_eval.c, all host threads) on a
bounded config sample of the same workload, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_REC = 1_000_000
N_MODELS = 4
LEVELS = 100
COST_RATIOS = (1.0, 4.0, 16.0, 64.0)
METRIC = "gear-plan config-evals/sec"
WORKLOAD = ("cfg2: Sentiment-140-shaped 4-stage cascade, 1M synthetic samples, binary scores, "
            "100-level grids, full cascade x threshold product")


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        out = {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
        if d.get("bf16_tflops"):
            out["bf16_tflops"] = float(d["bf16_tflops"])
        return out
    return {"hbm_gbs": 6650.0, "source": "fallback"}


def workload(seed: int = 0, device_grids: bool = True):
    """cfg2 inputs; grids from the device quantiles (gs_quantiles), or with
    numpy on the host for the reference arm (same values, bit for bit)."""
    from paper_2406_14424_b200 import synth
    profiles = synth.make_profiles(n_models=N_MODELS, cost_ratios=COST_RATIOS)
    cert, corr = synth.validation_matrices(N_MODELS, N_REC, 0.8, seed)
    if device_grids:
        from paper_2406_14424_b200.cascades import grid_values
    else:
        from oracle.oracle import grid_values
    grids = [np.array(grid_values(cert[:, j], LEVELS)) for j in range(N_MODELS)]
    return profiles, cert, corr, grids, profiles.cost1()


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples: list[list[str]] = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm = [float(s[0]) for s in self.samples if len(s) >= 7 and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) >= 7 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples if len(s) >= 7
                          for k in range(4) if "Active" in s[3 + k] and "Not" not in s[3 + k]})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def init_dist():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        # GS_ONE_DEVICE=1 + GS_DIST_BACKEND=gloo: every rank on cuda:0, for
        # exercising the sharded paths on a one-GPU box (not a measurement)
        dev_index = 0 if os.environ.get("GS_ONE_DEVICE") == "1" else local
        torch.cuda.set_device(dev_index)
        backend = os.environ.get("GS_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group(backend)
        local = dev_index
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    import torch
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


def max_over_ranks(x: float, world: int) -> float:
    import torch
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------------- ours -----
def run_ours(args, world, rank, local):
    import torch

    from oracle import oracle
    from paper_2406_14424_b200 import distributed as gdist
    from paper_2406_14424_b200.gridsweep import GridSweep, front_host, pareto_counts

    profiles, cert, corr, grids, cost1 = workload(seed=rank)  # one tenant per rank
    sw = GridSweep(cert, corr, grids, cost1, build=False)
    C = sw.n_configs
    L = sw.max_len
    dev = torch.device("cuda", torch.cuda.current_device())
    out = None
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2
    flush_read = torch.empty(512 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)

    def flush_l2():
        """Evict the L2 between timed steps: write 512 MB (> 126 MB L2); with
        --flush clean also read another 512 MB, so the L2 is left holding
        clean lines and the next step does not pay the write-back of the
        flush buffer's dirty lines (our data is evicted either way)."""
        if args.flush == "none":
            return
        flush.zero_()
        if args.flush == "clean":
            flush_read.sum()

    sw.build()
    out = sw.evaluate()
    # one step = one CUDA-graph launch (build + score every config)
    g_step = sw.capture(out)
    g_build = sw.capture(out, evaluate=False)
    g_eval = sw.capture(out, build=False)

    # warm-up
    for _ in range(args.warmup):
        g_step.replay()
    barrier(world)

    # timed: per-step CUDA events on the launching stream, L2 flushed between steps
    stream = torch.cuda.current_stream()

    def timed(graph, n):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(n)]
        for i in range(n):
            flush_l2()
            ev[i][0].record(stream)
            graph.replay()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in ev]

    # the timed step: one graph holding the L2 flush, then a start event
    # node, the sweep, an end event node -- the events bracket exactly the
    # sweep's kernels, with no graph-launch gap after the flush inside them
    ev_step = (torch.cuda.Event(enable_timing=True, external=True),
               torch.cuda.Event(enable_timing=True, external=True))
    g_timed = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_timed):
        flush_l2()
        ev_step[0].record()
        sw.build()
        sw.evaluate(out=out)
        ev_step[1].record()
    for _ in range(args.warmup):
        g_timed.replay()
    torch.cuda.synchronize()

    def timed_in_graph(n):
        res = []
        for _ in range(n):
            g_timed.replay()
            torch.cuda.synchronize()  # the event pair is re-recorded by the next replay
            res.append(ev_step[0].elapsed_time(ev_step[1]))
        return res

    with ClockSampler(local) as clocks:
        barrier(world)
        step_times = timed_in_graph(args.steps)
        barrier(world)
    step_ms = max_over_ranks(sum(step_times) / args.steps, world)
    # the previous protocol (stream events around a separate graph launch
    # after the flush): includes the GPU-side graph launch gap
    stream_ms = sum(timed(g_step, args.steps)) / args.steps
    value = world * C / (step_ms * 1e-3)
    build_ms = timed(g_build, args.steps)
    eval_ms = timed(g_eval, args.steps)
    part_ms = {}
    # the build's two passes: bucket sort + per-b1 planes (fast_path 2), or
    # histogram + plane pass (fast_path 1)
    names = ("g4_sort", "g4_gather") if sw.info.fast_path == 2 else ("g4_hist", "g4_plane")
    if sw.info.fast_path:
        # per-kernel durations inside the real step: external event-record
        # nodes between the three kernels of one captured step graph
        try:
            evs = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(4)]
            g_parts = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_parts):
                evs[0].record()
                sw.build(part="records")
                evs[1].record()
                sw.build(part="tables")
                evs[2].record()
                sw.evaluate(out=out)
                evs[3].record()
            acc = [0.0, 0.0, 0.0]
            for _ in range(args.steps):
                flush_l2()
                g_parts.replay()
                torch.cuda.synchronize()
                for k in range(3):
                    acc[k] += evs[k].elapsed_time(evs[k + 1])
            part_ms = {names[0]: acc[0] / args.steps, names[1]: acc[1] / args.steps,
                       "g4_eval": acc[2] / args.steps,
                       "timing": "event nodes inside the step graph (they also stop the "
                                 "programmatic launch overlap, so the parts sum above the step)"}
        except (RuntimeError, TypeError) as e:  # no timing events in graphs: one graph per kernel
            print(f"# per-kernel graph events unavailable ({e}); timing one graph per kernel",
                  file=sys.stderr)
            torch.cuda.synchronize()
            sw.build()
            g_rec = sw.capture(out, part="records")
            g_tab = sw.capture(out, part="tables")
            rec_t, tab_t = [], []
            for _ in range(args.steps):
                rec_t += timed(g_rec, 1)
                tab_t += timed(g_tab, 1)
            part_ms = {names[0]: sum(rec_t) / args.steps, names[1]: sum(tab_t) / args.steps,
                       "g4_eval": sum(eval_ms) / args.steps,
                       "timing": "one graph per kernel (includes graph launch)"}

    # correctness spot-check of the timed outputs (rank 0, sampled configs)
    check = None
    if rank == 0:
        rng = np.random.default_rng(1)
        pick = np.sort(rng.choice(C, size=64, replace=False))
        sm, thr, ns = oracle.grid_configs(grids)
        want = oracle.evaluate_encoded(cert, corr, sm[pick], thr[pick], ns[pick], cost1,
                                       n_threads=os.cpu_count() or 1)
        got_acc = out.accuracy.cpu().numpy()[pick]
        got_cost = out.mean_cost.cpu().numpy()[pick]
        got_frac = out.forward_frac.cpu().numpy()[pick]
        check = bool(np.array_equal(got_acc, want[0]) and np.array_equal(got_cost, want[1])
                     and np.array_equal(got_frac, want[2]))

    # ---- e2e through the public API from host buffers (+ front all-gather)
    pin_cert = torch.from_numpy(cert).pin_memory()
    pin_corr = torch.from_numpy(corr).pin_memory()
    dcert = torch.empty_like(pin_cert, device=dev)
    dcorr = torch.empty_like(pin_corr, device=dev)
    sw_e2e = GridSweep(dcert, dcorr, grids, cost1, build=False)
    e2e_out = None
    h2d = pin_cert.numel() * 8 + pin_corr.numel()
    d2h_total = 0

    def e2e_step():
        nonlocal e2e_out, d2h_total
        dcert.copy_(pin_cert, non_blocking=True)
        dcorr.copy_(pin_corr, non_blocking=True)
        sw_e2e.build()
        e2e_out = sw_e2e.evaluate(n_correct=True, out=e2e_out)
        idx = pareto_counts(e2e_out.n_correct, e2e_out.mean_cost, N_REC)
        front = gdist.gather_fronts(idx, e2e_out, world) if world > 1 else None
        rows = front_host(idx, e2e_out)  # one pinned D2H: [index, acc, cost, frac...]
        d2h_total = rows.nbytes + 8  # + the front size
        if front is not None:
            d2h_total += front.numel() * front.element_size()
        return rows

    e2e_pipelined = None
    if world == 1:
        # steady state of the public pipelined API: the H2D of set i+1 runs
        # while set i is swept and its front read back (SweepPipeline);
        # every step still copies its inputs in and its front rows out
        from paper_2406_14424_b200.pipeline import SweepPipeline
        pipe = SweepPipeline(N_REC, N_MODELS, grids, cost1, depth=3)
        for _ in range(args.warmup):
            pipe.submit(pin_cert, pin_corr)
        pipe.drain()
        torch.cuda.synchronize()
        tp = time.perf_counter()
        tickets = [pipe.submit(pin_cert, pin_corr) for _ in range(args.steps)]
        rows = [pipe.result(t) for t in tickets]
        torch.cuda.synchronize()
        e2e_pipelined = (time.perf_counter() - tp) * 1e3 / args.steps
        pipe_d2h = rows[-1].nbytes + 8
        del pipe
    for _ in range(args.warmup):
        e2e_step()
    barrier(world)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        flush_l2()  # same L2 state as the device-timed loop
        e2e_step()
    t1.record(stream)
    barrier(world)
    e2e_ms = max_over_ranks(t0.elapsed_time(t1) / args.steps, world)
    # subtract the flush (timed separately) so e2e counts only the sweep path
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        flush_l2()
    f1.record(stream)
    torch.cuda.synchronize()
    flush_ms = f0.elapsed_time(f1) / args.steps
    e2e_ms = max(e2e_ms - flush_ms, 1e-6)

    stage = None

    # ---- roofline for the dominant kernel (each kernel timed alone above)
    pk = peaks()
    b_in = N_REC * N_MODELS * 9
    b_out = C * (16 + 8 * L)
    build_avg = sum(build_ms) / args.steps
    eval_avg = sum(eval_ms) / args.steps
    alg_bytes = {names[0]: b_in, "g4_eval": b_out, "build": b_in, "eval": b_out}
    if part_ms:
        dom = max((names[0], "g4_eval"), key=lambda k: part_ms[k])
        dom_ms = part_ms[dom]
    else:
        dom, dom_ms = ("eval", eval_avg) if eval_avg >= build_avg else ("build", build_avg)
    dom_bytes = alg_bytes[dom]
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    step_gbs = (b_in + b_out) / (step_ms * 1e-3) / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "r2" / "traffic.json"
    if not tfile.exists():
        tfile = ROOT / "profiles" / "r1_traffic.json"
    if tfile.exists():
        traffic = json.loads(tfile.read_text()).get(dom)

    cfg4a = _guarded(config4a_bench, args, dev, world, rank) if not args.skip_config4a else None
    cpu = cpu_baseline(cert, corr, grids, cost1, args) if (rank == 0 and not args.no_cpu) else None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "config-evals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "ms_per_step_stream_events": stream_ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference make_validation semantics, default_rng(rank))",
            "config": {"workload": WORKLOAD, "n_records": N_REC, "n_models": N_MODELS,
                       "grid_levels": LEVELS, "n_configs_per_gpu": C,
                       "cost_ratios": list(COST_RATIOS),
                       "timing": "per step: one CUDA graph = 512 MB L2 flush, event node, "
                                 "sweep kernels, event node (events bracket the sweep only); "
                                 "ms_per_step_stream_events = events on the stream around a "
                                 "separate graph launch after the flush",
                       "l2": {"write": "flushed between timed steps: 512 MB write",
                              "clean": "flushed between timed steps: 512 MB write + 512 MB "
                                       "read (clean lines left)",
                              "none": "not flushed"}[args.flush], "parallelism": f"weak: 1 tenant sweep per GPU, "
                       f"NCCL all-gather of Pareto fronts in e2e ({world} ranks)"},
            "breakdown_ms": {"build": build_avg, "eval": eval_avg, **part_ms},
            "e2e": ({"value": C / (e2e_pipelined * 1e-3), "unit": "config-evals/s",
                     "ms_per_step": e2e_pipelined, "h2d_bytes_per_step": h2d,
                     "d2h_bytes_per_step": pipe_d2h,
                     "path": "SweepPipeline.submit/result from pinned host matrices: H2D of "
                             "set i+1 on a copy stream while set i is built, scored, reduced "
                             "to its exact Pareto front and the front rows read back; host "
                             "wall clock over the steps, synchronized on both sides",
                     "unpipelined": {"value": C / (e2e_ms * 1e-3), "ms_per_step": e2e_ms,
                                     "path": "GridSweep from pinned host matrices -> build "
                                             "-> eval -> pareto_counts -> D2H front rows"}}
                    if e2e_pipelined is not None else
                    {"value": world * C / (e2e_ms * 1e-3), "unit": "config-evals/s",
                     "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d,
                     "d2h_bytes_per_step": d2h_total,
                     "path": "GridSweep from pinned host matrices -> build -> eval -> "
                             "pareto_counts -> D2H front rows (+ NCCL all-gather of fronts)"}),
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved,
                         "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": achieved / pk["hbm_gbs"],
                         "traffic": traffic, "algorithmic_bytes": dom_bytes,
                         "kernel_ms": dom_ms,
                         "peak_source": pk["source"],
                         "step": {"bytes": b_in + b_out, "achieved": step_gbs,
                                  "frac": step_gbs / pk["hbm_gbs"]}},
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
            # per step, as gs_grid_plan reports them (gs_grid_info)
            "gpu_launches": args.steps * (sw.info.build_launches + sw.info.eval_launches),
            "fast_path": bool(sw.info.fast_path),
            "parity_spot_check": check,
        }
        if stage is not None:
            line["stage_step"] = stage
        # auxiliary legs never cost the headline line
        if not args.skip_ingest:
            line["ingest"] = _guarded(ingest_bench, args)
        if not args.skip_config4:
            line["config4b"] = _guarded(config4_bench, args, dev)
        if cfg4a is not None:
            line["config4a"] = cfg4a
        if not args.skip_config1:
            line["config1"] = _guarded(config1_bench, args, dev)
        if not args.skip_list:
            line["list_path"] = _guarded(list_path_bench, args, dev)
        if not args.skip_config3:
            line["config3"] = c3 = _guarded(config3_bench, args, dev)
            if "entropy" in c3:  # the online stage step at the config-3 shape
                line["stage_step"] = {k: c3[k]["stage_step"] for k in ("entropy", "margin")}
        if not args.skip_config5:
            line["config5"] = _guarded(config5_bench, args, dev)
        if not args.skip_head:
            line["head"] = _guarded(head_bench, args, dev)
        line["host"] = host_info()
        print(json.dumps(line), flush=True)


def _guarded(fn, *a):
    """Run an auxiliary bench leg; a failure is reported in the line, not raised."""
    try:
        return fn(*a)
    except Exception as e:  # noqa: BLE001
        import traceback
        traceback.print_exc(file=sys.stderr)
        return {"error": f"{type(e).__name__}: {e}"}


def config1_bench(args, dev):
    """BASELINE configs[0] (the reference's CPU default): a 3-model cascade,
    10k records, 100-level grids, the full product (C = 10,303) -- one CUDA
    graph per sweep (build + eval), L2 flushed between steps; launch-bound by
    design.  Beside it the oracle port of _evaluate_numba over all C configs
    on all host threads (the reference's own CPU default, 1 core, takes
    ~0.8 s: SURVEY 8d)."""
    import torch

    from oracle import oracle
    from paper_2406_14424_b200 import synth
    from paper_2406_14424_b200.cascades import grid_values
    from paper_2406_14424_b200.gridsweep import GridSweep
    profiles = synth.make_profiles()
    cert, corr = synth.validation_matrices(3, 10_000, 0.8, 0)
    grids = [np.array(grid_values(cert[:, j], LEVELS)) for j in range(3)]
    cost1 = profiles.cost1()
    sw = GridSweep(cert, corr, grids, cost1)
    out = sw.evaluate()
    g = sw.capture(out)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    for _ in range(3):
        g.replay()
    ts = []
    for _ in range(max(args.steps, 10)):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sum(ts) / len(ts)
    sm, thr, ns = oracle.grid_configs(grids)
    threads = os.cpu_count() or 1
    t = time.perf_counter()
    want = oracle.evaluate_encoded(cert, corr, sm, thr, ns, cost1, n_threads=threads)
    cpu_s = time.perf_counter() - t
    ok = bool(np.array_equal(out.accuracy.cpu().numpy(), want[0]) and
              np.array_equal(out.forward_frac.cpu().numpy(), want[2]))
    # stacked: R validation sets (seeds 0..R-1, each with its own device
    # quantile grids) swept by one gs_grid_sweep_batched launch
    from paper_2406_14424_b200.gridsweep import BatchedSweep
    R = 1024
    cs, ks, gs_ = [], [], []
    for seed in range(R):
        c, k = synth.validation_matrices(3, 10_000, 0.8, seed)
        cs.append(c)
        ks.append(k)
    cert_r = torch.from_numpy(np.stack(cs)).to(dev)
    corr_r = torch.from_numpy(np.stack(ks)).to(dev)
    for seed in range(R):
        gs_.append([np.array(grid_values(cert_r[seed, :, j], LEVELS)) for j in range(3)])
    glen = [min(len(g3[j]) for g3 in gs_) for j in range(3)]
    gs_ = [[g3[j][:glen[j]] for j in range(3)] for g3 in gs_]
    bs = BatchedSweep(cert_r, corr_r, gs_, cost1)
    res = bs.run()
    n_cfg_r = bs.n_configs
    for _ in range(3):
        bs.run()
    tb = []
    for _ in range(max(args.steps, 5)):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        bs.run()
        b.record()
        torch.cuda.synchronize()
        tb.append(a.elapsed_time(b))
    ms_r = sum(tb) / len(tb)
    # parity: a few stacked sets against their own single sweeps
    ok_r = True
    for seed in (0, 17, R - 1):
        one = GridSweep(cert_r[seed], corr_r[seed], gs_[seed], cost1).evaluate()
        ok_r = ok_r and bool(torch.equal(one.accuracy, res.accuracy[seed]) and
                             torch.equal(one.forward_frac, res.forward_frac[seed]))
    # e2e: the public API from pinned host matrices each step (H2D, build,
    # score every config, exact front, front rows D2H)
    from paper_2406_14424_b200.gridsweep import front_host
    pin_c = torch.from_numpy(cert).pin_memory()
    pin_k = torch.from_numpy(corr).pin_memory()
    dc, dk = torch.empty_like(pin_c, device=dev), torch.empty_like(pin_k, device=dev)
    sw_e = GridSweep(dc, dk, grids, cost1, build=False)
    e_out = None

    def e2e_step():
        nonlocal e_out
        dc.copy_(pin_c, non_blocking=True)
        dk.copy_(pin_k, non_blocking=True)
        sw_e.build()
        e_out = sw_e.evaluate(n_correct=True, out=e_out)
        idx, _ = sw_e.pareto(res=e_out)
        return front_host(idx, e_out)

    for _ in range(3):
        e2e_step()
    torch.cuda.synchronize()
    te = []
    for _ in range(max(args.steps, 10)):
        t = time.perf_counter()
        rows = e2e_step()
        te.append(time.perf_counter() - t)
    te.sort()
    e2e_ms = te[len(te) // 2] * 1e3
    b_r = R * (10_000 * 3 * 9 + n_cfg_r * (16 + 8 * 3))
    del flush, cert_r, corr_r, res, bs
    return {"workload": "cfg1: 3-model cascade, 10k records, 100-level grids, full product",
            "n_configs": sw.n_configs, "ms": ms, "config_evals_per_s": sw.n_configs / (ms * 1e-3),
            "launches_per_step": sw.info.build_launches + sw.info.eval_launches,
            "parity_full_product": ok,
            "e2e": {"value": sw.n_configs / (e2e_ms * 1e-3), "unit": "config-evals/s",
                    "ms_per_step": e2e_ms, "h2d_bytes_per_step": int(cert.nbytes + corr.nbytes),
                    "d2h_bytes_per_step": int(rows.nbytes),
                    "path": "GridSweep from pinned host matrices: H2D, build, eval, pareto, "
                            "front rows D2H; host wall clock, median"},
            "stacked": {"sets": R, "ms": ms_r, "config_evals_per_s": R * n_cfg_r / (ms_r * 1e-3),
                        "launches_per_step": 1, "algorithmic_bytes": b_r,
                        "achieved_gbs": b_r / (ms_r * 1e-3) / 1e9,
                        "frac": b_r / (ms_r * 1e-3) / 1e9 / peaks()["hbm_gbs"],
                        "parity_vs_single_sweeps": ok_r,
                        "path": "gridsweep.BatchedSweep.run (gs_grid_sweep_batched): one launch, a "
                                "CTA per set; seeds 0..R-1, per-set device quantile grids; L2 "
                                "flushed (512 MB write) before each step"},
            "cpu_baseline": {"value": sw.n_configs / cpu_s, "unit": "config-evals/s",
                             "cores": threads, "kind": "port",
                             "sample": "all 10,303 configs x 10k records (oracle/oracle_eval.c)"}}


def config4_bench(args, dev):
    """BASELINE configs[3] as variant 4b: a 5-stage cascade with
    100-level grids over 100k records, the full product (C = 105,101,005
    configs, 5.9 GB of reference-shaped outputs), one build + full eval
    (general path, gs_sweep.cu) per step; a sample of configs checked
    against the oracle walk."""
    import torch

    from oracle import oracle
    from paper_2406_14424_b200 import synth
    from paper_2406_14424_b200.cascades import grid_values
    from paper_2406_14424_b200.gridsweep import GridSweep
    m, n = 5, 100_000
    cert, corr = synth.validation_matrices(m, n, 0.8, 5)
    grids = [np.array(grid_values(cert[:, j], LEVELS)) for j in range(m)]
    cost1 = np.array([1.0, 4.0, 16.0, 64.0, 256.0])
    sw = GridSweep(cert, corr, grids, cost1, build=False)
    c = sw.n_configs
    out = None
    sw.build()
    out = sw.evaluate(out=out)
    times = []
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        sw.build()
        sw.evaluate(out=out)
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    ms = min(times)
    rng = np.random.default_rng(4)
    pick = np.sort(rng.choice(c, size=48, replace=False))
    sm, thr, ns = (t.cpu().numpy() for t in sw.decode(pick))
    want = oracle.evaluate_encoded(cert, corr, sm, thr, ns, cost1, n_threads=os.cpu_count() or 1)
    ok = bool(np.array_equal(out.accuracy[torch.from_numpy(pick).to(dev)].cpu().numpy(), want[0])
              and np.array_equal(out.mean_cost[torch.from_numpy(pick).to(dev)].cpu().numpy(),
                                 want[1]))
    threads = os.cpu_count() or 1
    pick_c = np.sort(rng.choice(c, size=threads * 16, replace=False))
    csm, cthr, cns = (t.cpu().numpy() for t in sw.decode(pick_c))
    t = time.perf_counter()
    oracle.evaluate_encoded(cert, corr, csm, cthr, cns, cost1, n_threads=threads)
    cpu_rate = len(pick_c) / (time.perf_counter() - t)
    out_bytes = c * (16 + 8 * m)
    gbs = (out_bytes + n * m * 9) / (ms * 1e-3) / 1e9
    del out
    torch.cuda.empty_cache()
    return {"workload": "cfg4b: 5-stage cascade, 100-level grids, 100k records, full product",
            "n_configs": c, "ms": ms, "config_evals_per_s": c / (ms * 1e-3),
            "algorithmic_bytes": out_bytes + n * m * 9, "achieved_gbs": gbs,
            "frac": gbs / peaks()["hbm_gbs"], "fast_path": bool(sw.info.fast_path),
            "parity_spot_check": ok, "timing": "best of 3 (build + full eval), no L2 flush "
                                               "(5.9 GB of outputs per step)",
            "cpu_baseline": {"value": cpu_rate, "unit": "config-evals/s", "cores": threads,
                             "kind": "port", "sample": f"{len(pick_c)} random configs x 100k "
                                                       "records, oracle/oracle_eval.c"}}


def ingest_bench(args, n=200_000):
    """Validation ingest: a reference-format JSONL of n
    records (4 models, binary scores) -> device certainty/correct matrices
    through formats.load_validation_arrays (native multi-threaded reader +
    gs_certainty), against the reference reader restated in
    oracle.load_validation_jsonl on a 20k-line slice (one core, as shipped)."""
    import tempfile

    import torch

    from oracle import oracle
    from paper_2406_14424_b200 import formats, synth
    from paper_2406_14424_b200.cascades import _device_matrices
    profiles = synth.make_profiles(n_models=N_MODELS, cost_ratios=COST_RATIOS)
    va = synth.binary_logit_arrays(profiles, n, 0.8, seed=11, dtype=np.float64)
    ids = profiles.model_ids
    tmp = Path(tempfile.mkdtemp())
    path, sample = tmp / "v.jsonl", tmp / "s.jsonl"
    sc = [va.scores[m] for m in ids]
    with open(path, "w") as f:
        for i in range(n):
            parts = ", ".join(f'"{m}": {{"scores": [{float(sc[j][i, 0])!r}, {float(sc[j][i, 1])!r}], '
                              f'"correct": {"true" if va.correct[i, j] else "false"}}}'
                              for j, m in enumerate(ids))
            f.write(f'{{"sample_id": {i}, "models": {{{parts}}}}}\n')
    with open(path) as f, open(sample, "w") as g:
        for _, line in zip(range(20_000), f):
            g.write(line)
    size = path.stat().st_size
    best = None
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        arr = formats.load_validation_arrays(path)
        cert, corr = _device_matrices(arr, profiles)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        best = dt if best is None else min(best, dt)
    t = time.perf_counter()
    oracle.load_validation_jsonl(sample)
    ref_dt = time.perf_counter() - t
    for p in (path, sample):
        p.unlink()
    tmp.rmdir()
    return {"records_per_s": n / best, "ms": best * 1e3, "file_mb": size / 1e6,
            "path": "formats.load_validation_arrays (gs_jsonl_* all host threads) -> "
                    "device certainty (gs_certainty) + correct matrices",
            "cpu_baseline": {"records_per_s": 20_000 / ref_dt, "cores": 1, "kind": "port",
                             "sample": "20k lines, oracle.load_validation_jsonl (json.loads "
                                       "per line, src/formats.py:75-97)"}}


def host_info() -> dict:
    """CPU model, logical cores and this process's affinity."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except AttributeError:
        aff = os.cpu_count()
    return {"cpu_model": model, "cpu_count": os.cpu_count(), "affinity": aff}


def _ref_gearserve():
    """The unmodified reference from baseline/_ref (tools/install_reference.sh)
    when it travelled with the snapshot and numba imports; else None."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "gearserve").is_dir():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/gs_numba_cache")
    if str(ref) not in sys.path:
        sys.path.append(str(ref))
    try:
        from gearserve import kernels as ref_kernels
        return ref_kernels
    except Exception:  # noqa: BLE001
        return None


def list_path_bench(args, dev):
    """The operator the reference exposes, kernels.evaluate_encoded (list
    path, gs_eval_encoded), at (a) the reference's published benchmark point
    (bench_kernels.py: records=4000 models=6 cascades=200; numba 5.3 ms,
    numpy 17.0 ms on one core, README.md:131-135) through the numpy-in /
    numpy-out drop-in, and (b) SP1's shape: 2000 sampled cascades
    (sample_cascades over the cfg2 100-level grids) x 1M records, device
    resident.  CPU: the oracle port on one core (a) / all cores (b), and the
    reference's own numba walk when baseline/_ref is present."""
    import torch

    from oracle import oracle
    from paper_2406_14424_b200 import kernels, synth
    from paper_2406_14424_b200.cascades import encode_cascades, sample_cascades
    from paper_2406_14424_b200.cascades import ThresholdGrid

    out = {}
    prob = synth.kernels_bench_problem(4000, 6, 200, 0)
    got = kernels.evaluate_encoded(*prob)
    want = oracle.evaluate_encoded(*prob, n_threads=1)
    ok = all(np.array_equal(a, b) for a, b in zip(got, want))
    ts = []
    for _ in range(max(args.steps, 10)):
        t = time.perf_counter()
        kernels.evaluate_encoded(*prob)
        ts.append(time.perf_counter() - t)
    ts.sort()
    dev_args = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in prob]
    for _ in range(3):
        kernels.evaluate_encoded_device(*dev_args)
    a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = max(args.steps, 10)
    a_ev.record()
    for _ in range(k):
        kernels.evaluate_encoded_device(*dev_args)
    b_ev.record()
    torch.cuda.synchronize()
    dev_ms = a_ev.elapsed_time(b_ev) / k
    t = time.perf_counter()
    for _ in range(5):
        oracle.evaluate_encoded(*prob, n_threads=1)
    port_ms = (time.perf_counter() - t) / 5 * 1e3
    pub = {"records": 4000, "models": 6, "cascades": 200,
           "e2e_ms_median": ts[len(ts) // 2] * 1e3, "e2e_ms_best": ts[0] * 1e3,
           "device_ms": dev_ms, "bit_exact_vs_oracle": ok,
           "published_numba_ms": 5.3, "published_numpy_ms": 17.0,
           "e2e_speedup_vs_published_numba": 5.3 / (ts[len(ts) // 2] * 1e3),
           "path": "kernels.evaluate_encoded: numpy in (H2D), gs_eval_encoded, numpy out (D2H); "
                   "device_ms = evaluate_encoded_device on resident tensors (CUDA events)",
           "cpu_baseline": {"value": port_ms, "unit": "ms/call", "cores": 1, "kind": "port",
                            "sample": "the whole problem, oracle/oracle_eval.c, 1 thread"}}
    ref = _ref_gearserve()
    if ref is not None and getattr(ref, "HAS_NUMBA", False):
        ref._evaluate_numba(*prob)  # JIT / cache load
        t = time.perf_counter()
        for _ in range(5):
            r = ref._evaluate_numba(*prob)
        pub["reference_numba"] = {"value": (time.perf_counter() - t) / 5 * 1e3, "unit": "ms/call",
                                  "cores": 1, "kind": "reference",
                                  "bit_exact": all(np.array_equal(x, y) for x, y in zip(r, got)),
                                  "sample": "baseline/_ref gearserve.kernels._evaluate_numba, as shipped"}
    out["published_point"] = pub

    # (b) SP1 shape: 2000 sampled cascades x the cfg2 records
    profiles, cert, corr, grids, cost1 = workload(seed=0)
    grid = ThresholdGrid({m: tuple(float(x) for x in grids[j])
                          for j, m in enumerate(profiles.model_ids)})
    cascs = sample_cascades(profiles, grid, 2000, rng_seed=0)
    sm, thr, ns = encode_cascades(cascs, profiles)
    dcert = torch.from_numpy(cert).to(dev)
    dcorr = torch.from_numpy(corr).to(dev)
    dsm, dthr, dns = (torch.from_numpy(x).to(dev) for x in (sm, thr, ns))
    dcost = torch.from_numpy(cost1).to(dev)
    kernels.evaluate_encoded_device(dcert, dcorr, dsm, dthr, dns, dcost)
    a_ev.record()
    for _ in range(3):
        r = kernels.evaluate_encoded_device(dcert, dcorr, dsm, dthr, dns, dcost)
    b_ev.record()
    torch.cuda.synchronize()
    sp1_ms = a_ev.elapsed_time(b_ev) / 3
    pick = np.arange(0, len(cascs), max(1, len(cascs) // 64))
    threads = os.cpu_count() or 1
    t = time.perf_counter()
    want = oracle.evaluate_encoded(cert, corr, sm[pick], thr[pick], ns[pick], cost1,
                                   n_threads=threads)
    cpu_dt = time.perf_counter() - t
    ok_b = bool(np.array_equal(r[0].cpu().numpy()[pick], want[0]) and
                np.array_equal(r[2].cpu().numpy()[pick], want[2]))
    steps = int(ns.astype(np.int64).sum())  # upper bound of stage visits per record
    out["sp1_shape"] = {
        "cascades": len(cascs), "records": N_REC, "device_ms": sp1_ms,
        "config_evals_per_s": len(cascs) / (sp1_ms * 1e-3),
        "record_config_pairs_per_s": len(cascs) * N_REC / (sp1_ms * 1e-3),
        "bound": "issue (O(C*N*stages) walk: one thread per cascade, records broadcast from "
                 "shared memory; the HBM bytes are N*M*9 = 36 MB, ~6 us)",
        "stage_visits_upper_bound": steps * N_REC,
        "parity_spot_check": ok_b,
        "cpu_baseline": {"value": len(pick) / cpu_dt, "unit": "config-evals/s", "cores": threads,
                         "kind": "port",
                         "sample": f"{len(pick)} of the {len(cascs)} cascades x 1M records, "
                                   "oracle/oracle_eval.c"}}
    del dcert, dcorr
    return out


def config3_bench(args, dev):
    """BASELINE configs[2]: an ImageNet-shaped 3-model cascade (ResNet-
    18/50/152 stand-ins), 1M samples, 1000-class f32 logits per model
    (synth.imagenet_logits; correct = argmax == label).  One step: the
    certainty of every logit row of the three models (entropy, the config's
    named kind; margin = the reference's Eq. 5) into the [N, 3] matrix, the
    device quantile grids (levels 100), the full grid sweep (C = 10,303) and
    its exact Pareto front.  Beside it the stage step at thresholds chosen at
    the 35th certainty percentile (so about a third of the rows defer and
    compaction runs), and the reference's certainty on the CPU."""
    import torch

    from oracle import oracle
    from paper_2406_14424_b200 import synth
    from paper_2406_14424_b200.cascades import certainty_rows, grid_values
    from paper_2406_14424_b200.gridsweep import GridSweep
    from paper_2406_14424_b200.stage import stage_step

    n, n_cls, m = N_REC, 1000, 3
    logits, _, labels = synth.imagenet_logits(n, n_cls, m, seed=0, device=dev)
    corr = torch.stack([(x.argmax(dim=1) == labels).to(torch.uint8) for x in logits], 1)
    corr = corr.contiguous()
    cost1 = np.array([1.8, 4.1, 11.5]) * 1000.0  # ResNet-18/50/152 GFLOP ratios, µs
    pk = peaks()
    out = {"workload": "cfg3: 3 x [1M, 1000] f32 logits (ResNet-18/50/152 stand-ins), "
                       "certainty -> [N,3] matrices -> 100-level device grids -> full sweep "
                       "(C = 10,303) -> exact Pareto front",
           "correct": "argmax(logits) == label (setup, untimed)"}
    for kind in ("entropy", "margin"):
        def step():
            cert = torch.stack([certainty_rows(x, kind=kind) for x in logits], 1).contiguous()
            grids = [grid_values(cert[:, j], LEVELS) for j in range(m)]
            sw = GridSweep(cert, corr, grids, cost1)
            idx, res = sw.pareto()
            return cert, sw, idx, res
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        ts = []
        for _ in range(max(3, min(args.steps, 5))):
            t = time.perf_counter()
            cert, sw, idx, res = step()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t)
        ms = min(ts) * 1e3
        # certainty phase alone (the bytes: the logits), CUDA events
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_ev.record()
        for x in logits:
            certainty_rows(x, kind=kind)
        b_ev.record()
        torch.cuda.synchronize()
        cert_ms = a_ev.elapsed_time(b_ev)
        bytes_ = m * n * (n_cls * 4 + 8)
        gbs = bytes_ / (cert_ms * 1e-3) / 1e9
        # parity: the sweep against the oracle walk on sampled configs,
        # certainty against the f64 numpy oracle on sampled rows
        rng = np.random.default_rng(3)
        rows = np.sort(rng.choice(n, 2000, replace=False))
        lg = [x[torch.from_numpy(rows).to(dev)].cpu().numpy() for x in logits]
        fn = oracle.entropy_rows if kind == "entropy" else oracle.margin_rows
        c_ref = np.stack([fn(z) for z in lg], 1)
        c_got = cert.cpu().numpy()[rows]
        cert_ok = bool(np.max(np.abs(c_got - c_ref)) <= 5e-7) if kind == "entropy" else \
            bool(np.array_equal(c_got, c_ref))
        pick = np.sort(rng.choice(sw.n_configs, 64, replace=False))
        sm, thr, ns = (t.cpu().numpy() for t in sw.decode(pick))
        want = oracle.evaluate_encoded(cert.cpu().numpy(), corr.cpu().numpy(), sm, thr, ns, cost1,
                                       n_threads=os.cpu_count() or 1)
        sweep_ok = bool(np.array_equal(res.accuracy.cpu().numpy()[pick], want[0]))
        out[kind] = {"ms_per_step": ms, "logit_rows_per_s": m * n / (ms * 1e-3),
                     "certainty_ms": cert_ms, "certainty_rows_per_s": m * n / (cert_ms * 1e-3),
                     "certainty_roofline": {"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"],
                                            "unit": "GB/s", "frac": gbs / pk["hbm_gbs"],
                                            "algorithmic_bytes": bytes_},
                     "front_size": int(idx.numel()), "n_configs": sw.n_configs,
                     "certainty_check": cert_ok, "sweep_spot_check": sweep_ok,
                     "timing": "host wall clock around the synchronized pipeline, best of "
                               f"{len(ts)}; certainty_ms by CUDA events"}
        # stage step of model 0 at its 35th certainty percentile
        thr_v = float(np.quantile(cert[:, 0].cpu().numpy(), 0.35))
        thr_t = torch.full((n,), thr_v, dtype=torch.float64, device=dev)
        for _ in range(2):
            r = stage_step(logits[0], thr_t, kind=kind, sync=False)
        a_ev.record()
        for _ in range(5):
            r = stage_step(logits[0], thr_t, kind=kind, sync=False)
        b_ev.record()
        torch.cuda.synchronize()
        st_ms = a_ev.elapsed_time(b_ev) / 5
        d = int(r.counts[0].item())
        b_st = n * n_cls * 4 + n * (8 + 1) + d * 8
        out[kind]["stage_step"] = {
            "ms": st_ms, "samples_per_s": n / (st_ms * 1e-3), "threshold": thr_v, "deferred": d,
            "deferred_frac": d / n, "algorithmic_bytes": b_st,
            "frac": b_st / (st_ms * 1e-3) / 1e9 / pk["hbm_gbs"]}
    # e2e: logits from pinned host memory (H2D inside the timed region),
    # certainty + sweep + front, the front rows read back
    out["e2e"] = _guarded(config3_e2e, logits, corr, cost1, dev)
    # CPU: the reference's certainty (sorted() per row, src/cascades.py:20-28)
    # on 2000 rows, and f64 numpy margin / entropy on 50k rows, one core
    lg0 = logits[0][:50_000].cpu().numpy()
    t = time.perf_counter()
    for i in range(2000):
        oracle.certainty(lg0[i].tolist())
    ref_rate = 2000 / (time.perf_counter() - t)
    t = time.perf_counter()
    oracle.margin_rows(lg0)
    np_margin = 50_000 / (time.perf_counter() - t)
    t = time.perf_counter()
    oracle.entropy_rows(lg0)
    np_entropy = 50_000 / (time.perf_counter() - t)
    out["cpu_baseline"] = {"value": ref_rate, "unit": "rows/s", "cores": 1, "kind": "port",
                           "sample": "2000 rows of model 0: cascades.certainty semantics "
                                     "(sorted per row, oracle.certainty)",
                           "numpy_f64_margin_rows_per_s": np_margin,
                           "numpy_f64_entropy_rows_per_s": np_entropy}
    del logits
    torch.cuda.empty_cache()
    return out


def config3_e2e(logits, corr, cost1, dev):
    """Config 3 end to end from HOST logits: pinned [N, 1000] f32 per model,
    streamed to the device in row chunks on a copy stream while the previous
    chunk's certainty runs, then grids, sweep, front, front rows to host."""
    import psutil
    import torch

    from paper_2406_14424_b200.cascades import certainty_rows, grid_values
    from paper_2406_14424_b200.gridsweep import GridSweep, front_host

    n, n_cls = logits[0].shape
    need = len(logits) * n * n_cls * 4
    if psutil.virtual_memory().available < 3 * need:
        return {"skipped": f"host memory: {psutil.virtual_memory().available / 1e9:.0f} GB free"}
    host = [torch.empty((n, n_cls), dtype=torch.float32, pin_memory=True) for _ in logits]
    for h, x in zip(host, logits):
        h.copy_(x)
    chunk = 65536
    bufs = [torch.empty((chunk, n_cls), dtype=torch.float32, device=dev) for _ in range(2)]
    copy = torch.cuda.Stream()
    main = torch.cuda.current_stream()
    cert = torch.empty((n, len(logits)), dtype=torch.float64, device=dev)
    evs = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]

    def step():
        k = 0
        for j, h in enumerate(host):
            for lo in range(0, n, chunk):
                hi = min(n, lo + chunk)
                b = k % 2
                with torch.cuda.stream(copy):
                    copy.wait_event(free[b])
                    bufs[b][: hi - lo].copy_(h[lo:hi], non_blocking=True)
                    evs[b].record(copy)
                main.wait_event(evs[b])
                cert[lo:hi, j] = certainty_rows(bufs[b][: hi - lo], kind="entropy")
                free[b].record(main)
                k += 1
        c = cert.contiguous()
        grids = [grid_values(c[:, j], LEVELS) for j in range(len(host))]
        sw = GridSweep(c, corr, grids, cost1)
        idx, res = sw.pareto()
        return front_host(idx, res)

    step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        rows = step()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    ms = min(ts) * 1e3
    return {"ms_per_step": ms, "logit_rows_per_s": len(host) * n / (ms * 1e-3),
            "h2d_bytes_per_step": need, "d2h_bytes_per_step": int(rows.nbytes),
            "path": "pinned host logits -> 64k-row chunks H2D on a copy stream overlapped with "
                    "certainty_rows (entropy) -> grid_values -> GridSweep.pareto -> front_host; "
                    "host wall clock, best of 3"}


def config4a_bench(args, dev, world, rank):
    """BASELINE configs[3] as variant 4a: 5 models, 1000-level
    device-quantile grids, 100k records, the full cascade m0 -> .. -> m4 over
    every threshold tuple -- g0 g1 g2 g3 = 1.0e12 configs -- reduced to its
    exact Pareto front (front5.py / gs_front5.cu: two streaming passes, no
    per-config output).  Sharded by k0 over the ranks (strong scaling): pass 1
    on each rank's k0 slice, an NCCL all-reduce (MIN) of the per-accuracy
    minimum costs, pass 2 on the slice, an all-reduce of the per-point tie
    counts (SUM) and smallest indices (MIN).  The front of 1000-level grids
    holds ~1e9 tied configs (threshold tuples that route every record alike:
    e.g. k0 = 0 stops every record at m0), so it is reported as its distinct
    points with their tie counts and smallest config index.  CPU: the oracle
    walk on 4,096 random configs of the full cascade x 100k records."""
    import torch

    from oracle import oracle
    from paper_2406_14424_b200 import synth
    from paper_2406_14424_b200.cascades import grid_values
    from paper_2406_14424_b200.front5 import Front5
    n = 100_000
    cert, corr = synth.validation_matrices(5, n, 0.8, 7)
    grids = [np.array(grid_values(cert[:, j], 1000)) for j in range(5)]
    cost1 = np.array([1.0, 4.0, 16.0, 64.0, 256.0])
    f5 = Front5(cert, corr, grids, cost1)
    cuts = f5.k0_cuts(world)  # about equal work per rank (a k0's cost grows with #(b0 <= k0))
    b, e = int(cuts[rank]), int(cuts[rank + 1])

    def step():
        f5.prepare()
        f5.pass1(b, e)
        if world > 1:
            import torch.distributed as dist
            dist.all_reduce(f5.mincost(), op=dist.ReduceOp.MIN)
        f5.select()
        f5.pass2(b, e, cap=0)
        if world > 1:
            import torch.distributed as dist
            ties = f5._ws_view(int(f5.info.ties_offset))
            mi = f5._ws_view(int(f5.info.min_index_offset))
            dist.all_reduce(ties, op=dist.ReduceOp.SUM)
            mi_signed = mi.clone()
            mi_signed[mi_signed < 0] = torch.iinfo(torch.int64).max  # 0xff.. = none
            dist.all_reduce(mi_signed, op=dist.ReduceOp.MIN)
            mi.copy_(mi_signed)
        torch.cuda.synchronize()

    barrier(world)
    t = time.perf_counter()
    step()
    barrier(world)
    sec = max_over_ranks(time.perf_counter() - t, world)
    if rank != 0:
        return None
    acc_cnt, cost, ties, mi = f5.points()
    # spot check: the cheapest and the most accurate front points' smallest
    # configs against the oracle walk
    chk = np.unique(np.concatenate([mi[:3], mi[-3:]]).astype(np.int64))
    sm, thr, ns = f5.decode(chk)
    want = oracle.evaluate_encoded(cert, corr, sm, thr, ns, cost1, n_threads=os.cpu_count() or 1)
    pos = {int(m): k for k, m in enumerate(mi)}
    ok = all(want[0][q] == acc_cnt[pos[int(c)]] / n and want[1][q] == cost[pos[int(c)]]
             for q, c in enumerate(chk))
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(4)
    pick = np.sort(rng.choice(f5.n_configs, size=4096, replace=False))
    csm, cthr, cns = f5.decode(pick)
    t = time.perf_counter()
    oracle.evaluate_encoded(cert, corr, csm, cthr, cns, cost1, n_threads=threads)
    cpu_rate = len(pick) / (time.perf_counter() - t)
    return {"workload": "cfg4a: 5-stage cascade, 1000-level device-quantile grids, 100k records, "
                        "the full cascade's every threshold tuple, exact Pareto front",
            "grid_len": f5.grid_len, "n_configs": f5.n_configs, "seconds": sec,
            "config_evals_per_s": f5.n_configs / sec, "gpus": world,
            "scaling": "strong: k0 sharded over the ranks, NCCL all-reduce (MIN) of the per-"
                       "accuracy minimum costs between the passes",
            "front_points": int(len(acc_cnt)), "front_configs": int(ties.sum()),
            "front_accuracy_range": [float(acc_cnt.min() / n), float(acc_cnt.max() / n)],
            "front_cost_range": [float(cost.min()), float(cost.max())],
            "spot_check_vs_oracle": bool(ok),
            "bound": "issue (staircase scoring of 1e12 configs from per-row b3 histograms; "
                     "records stream from L2; no per-config HBM traffic)",
            "cpu_baseline": {"value": cpu_rate, "unit": "config-evals/s", "cores": threads,
                             "kind": "port", "sample": "4,096 random configs of the full cascade "
                                                       "x 100k records, oracle/oracle_eval.c"}}


def head_bench(args, dev, B=262_144, N=1000, K=2048):
    """A cascade stage's classifier head on the tensor cores fused with its
    certainty (gs_head_certainty): ResNet-50-shaped head (2048 features ->
    1000 classes), bf16 features and weight, f32 accumulation in TMEM, entropy
    certainty per row.  CUDA events around back-to-back calls (the 1 GB of
    features exceeds L2); beside it the unfused path (cuBLAS bf16 GEMM ->
    logits -> gs_certainty).  Parity: the first 4096 rows vs a float64 torch
    reference of the same op."""
    import math
    import torch

    from paper_2406_14424_b200.cascades import certainty_rows
    from paper_2406_14424_b200.head import head_certainty

    g = torch.Generator(device=dev).manual_seed(7)
    f = torch.randn(B, K, device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device=dev, generator=g) / math.sqrt(K) * 3).to(torch.bfloat16)
    bias = torch.randn(N, device=dev, generator=g) * 0.1

    def timed(fn, reps=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    ms = timed(lambda: head_certainty(f, w, bias, kind="entropy"))
    ms_unfused = timed(lambda: certainty_rows(f @ w.T + bias, kind="entropy"))
    cert = head_certainty(f[:4096], w, bias, kind="entropy")
    x = f[:4096].double() @ w.double().T + bias.double()
    p = torch.softmax(x, dim=1)
    ref = 1.0 - (-(p * torch.log_softmax(x, dim=1)).sum(dim=1)) / math.log(N)
    err = float((cert - ref).abs().max())
    flops = 2.0 * B * N * K
    tf = flops / (ms * 1e-3) / 1e12
    pk = peaks()
    peak = pk.get("bf16_tflops") or 2250.0
    return {"workload": f"classifier head + entropy certainty: features [{B}, {K}] bf16 x weight [{N}, {K}] "
                        "bf16 (+ f32 bias) -> f64 certainty per row; logits never stored",
            "ms": ms, "rows_per_s": B / (ms * 1e-3), "tflops": tf,
            "roofline": {"bound": "tensor", "achieved": tf, "peak": peak, "unit": "TFLOP/s",
                         "frac": tf / peak,
                         "peak_source": "measured" if pk.get("bf16_tflops") else "nominal"},
            "unfused": {"ms": ms_unfused, "tflops": flops / (ms_unfused * 1e-3) / 1e12,
                        "path": "torch bf16 matmul (cuBLAS) + bias -> bf16 logits -> certainty_rows"},
            "max_abs_err_vs_f64": err, "parity_ok": err < 2e-5,
            "timing": "CUDA events around 10 back-to-back calls after 3 warm-up calls"}


def online_router_bench(plan, prof, cert, corr):
    """The live-serving shape of the stage step: StageRouter.finish_batch
    (EngineState.finish_batch, src/engine.py:355-383) on batches of 4 / 8 /
    64 / 1024 items -- one packed H2D, the device gate, one packed D2H, the
    host's replica draws and queue appends per call -- against the
    reference's loop restated (oracle.finish_batch) on the same batches,
    one core.  At 4-8 items a call is latency-bound (one round trip)."""
    from oracle import oracle
    from paper_2406_14424_b200.engine import GearTables, Item, StageRouter
    reps = list(plan.placement.replicas)
    ids = list(prof.model_ids)
    devs = []
    for r in reps:
        if r.device_id not in devs:
            devs.append(r.device_id)
    tables = GearTables.from_gears(plan.gears, [(r.replica_id, r.model_id) for r in reps],
                                   {m: j for j, m in enumerate(ids)})
    gears_o = [{"stage_model": tables.stage_models[g], "thresholds": tables.thresholds[g],
                "replica_idx": tables.replicas[g], "cum_weights": tables.cum_weights[g]}
               for g in range(len(plan.gears))]
    rng = np.random.default_rng(0)
    out = {}
    for bsz in (4, 8, 64, 1024):
        n_calls = max(20, 40_000 // bsz)
        batches = []
        for c in range(n_calls):
            g = rng.integers(0, len(plan.gears), bsz)
            st = np.array([int(rng.integers(0, len(tables.stage_models[x]))) for x in g])
            rows = rng.integers(0, cert.shape[0], bsz)
            batches.append([(int(c * bsz + k), int(rows[k]), int(st[k]), int(g[k])) for k in range(bsz)])
        router = StageRouter(tables, cert, corr, [devs.index(r.device_id) for r in reps], seed=0)
        for b in batches[:3]:
            router.finish_batch(0, [Item(i, r, s_, g_, 0) for i, r, s_, g_ in b], 10)
        t = time.perf_counter()
        for b in batches:
            router.finish_batch(0, [Item(i, r, s_, g_, 0) for i, r, s_, g_ in b], 10)
        dev_rate = n_calls * bsz / (time.perf_counter() - t)
        orng = np.random.default_rng(0)
        t = time.perf_counter()
        for b in batches:
            oracle.finish_batch([{"request_id": i, "row": r, "stage": s_, "gear": g_, "arrival_us": 0}
                                 for i, r, s_, g_ in b], gears_o, cert, corr, orng, 10)
        cpu_rate = n_calls * bsz / (time.perf_counter() - t)
        out[f"batch_{bsz}"] = {"samples_per_s": dev_rate, "calls": n_calls,
                               "cpu_baseline_samples_per_s": cpu_rate}
    out["path"] = ("StageRouter.finish_batch: Item objects in, packed pinned H2D, gs_stage_gate_packed "
                   "(one tile), packed pinned D2H, replica draws (Python lists up to 256 items, numpy above), deque appends; host "
                   "wall clock. cpu_baseline: oracle.finish_batch (the reference loop restated), "
                   "1 core")
    return out


def config5_bench(args, dev):
    """BASELINE configs[4]: an Azure-like bursty trace (20 min of lognormal
    per-second levels, default_rng(0), scaled to 7,600 max QPS with
    formats.scale_trace semantics: 1.32M requests) replayed through the
    serving engine -- batched routing, the certainty gate, gear switching
    every 100 ms -- by 8 independent replica groups (synth.replica_group_plan,
    request i -> group i % 8), each one engine.run (virtual clock) on the
    device: replay.run_many, one launch, one warp per group.  The replay is a
    sequential event loop per group, so a group runs on one warp; the GPU's
    width goes to independent groups and probes (the `probes` sub-leg: 1,024
    SP1 burst-throughput probes, src/planner.py:329-357, in one launch).
    CPU: the reference engine loop (oracle.engine_run restatement, and the
    shipped reference from baseline/_ref when present) on a bounded prefix of
    group 0's trace, one core; parity: that prefix's records, device vs CPU."""
    import torch

    from oracle import oracle
    from paper_2406_14424_b200 import replay, synth
    from paper_2406_14424_b200.types import (Cascade, Gear, GearPlan, ValidationArrays,
                                             WorkloadTrace)
    groups = 8
    trace = replay.scale_trace(synth.trace_from_counts(synth.bursty_counts(1200, 0)), 7600.0)
    parts = replay.split_round_robin(trace, groups)
    prof, plan = synth.replica_group_plan(qps_max=7600.0 / groups)
    cert, corr = synth.validation_matrices(4, 100_000, 0.8, 5)
    val = ValidationArrays(prof.model_ids, certainty=cert, correct=corr)
    dp = replay.DevicePlan(plan, prof, val)
    cfg = replay.EngineConfig(seed=0)
    jobs = [replay.Job(dp, p.arrivals, p.duration_us, replay.EngineConfig(seed=g))
            for g, p in enumerate(parts)]
    prep = replay.Prepared(jobs)
    prep.run()  # warm
    torch.cuda.synchronize()
    a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a_ev.record()
    prep.run()  # one launch: every group's event loop
    b_ev.record()
    torch.cuda.synchronize()
    ms = a_ev.elapsed_time(b_ev)
    res = prep.results()
    done = sum(r.completed for r in res)
    routed = sum(int(r.records["stages_executed"].sum()) for r in res)
    gear_hist = np.bincount(np.concatenate([r.windows["gear_after"] for r in res]), minlength=4)
    t = time.perf_counter()
    replay.run_many(jobs)
    e2e_ms = (time.perf_counter() - t) * 1e3
    out = {"workload": "cfg5: 20-min bursty trace scaled to 7,600 max QPS (1.32M requests), "
                       "8 replica groups x (4-model cascade on 4 devices, 4 gears), "
                       "engine.run virtual clock per group",
           "requests": len(trace), "groups": groups, "ms": ms,
           "requests_per_s": len(trace) / (ms * 1e-3),
           "routed_samples_per_s": routed / (ms * 1e-3), "completed": done,
           "gear_windows": gear_hist.tolist(),
           "e2e": {"ms": e2e_ms, "value": routed / (e2e_ms * 1e-3), "unit": "routed samples/s",
                   "path": "replay.run_many: plan tables + traces H2D, one launch, records / "
                           "windows / counters D2H; host wall clock"},
           "launches": 1, "bound": "latency: one sequential event loop per group (warp)"}
    # CPU: the reference engine loop on a prefix of group 0, one core
    n_cpu = 60_000
    sub = WorkloadTrace(parts[0].arrivals[:n_cpu],
                        duration_us=int(parts[0].arrivals[n_cpu - 1]) // 1_000_000 * 1_000_000 +
                        1_000_000)
    ids = list(prof.model_ids)
    runtime = [[0] + [prof[m].runtime_us(b) for b in range(1, 9)] for m in ids]
    t = time.perf_counter()
    ref = oracle.engine_run(plan, sub, cert, corr, runtime, [8] * 4,
                            {m: j for j, m in enumerate(ids)}, seed=0)
    cpu_s = time.perf_counter() - t
    dev_sub = replay.run_many([replay.Job(dp, sub.arrivals, sub.duration_us, cfg)])[0]
    r = dev_sub.records
    got = np.stack([r["request_id"], dev_sub.arrival_us[r["request_id"]], r["completion_us"],
                    r["stages_executed"], r["correct"], r["gear_index"]], 1).astype(np.int64)
    routed_cpu = int(ref["records"][:, 3].sum())
    out["parity_prefix"] = bool(np.array_equal(got, ref["records"]))
    out["cpu_baseline"] = {"value": routed_cpu / cpu_s, "unit": "routed samples/s", "cores": 1,
                           "kind": "port", "requests_per_s": n_cpu / cpu_s,
                           "sample": f"first {n_cpu} requests of group 0, oracle.engine_run "
                                     "(engine.run's loop restated), one core"}
    refmod = _ref_gearserve()
    if refmod is not None:
        try:
            from gearserve import engine as reng
            from gearserve import types as rt
            rplan = rt.GearPlan(
                placement=rt.Placement([rt.Replica(x.replica_id, x.model_id, x.device_id)
                                        for x in plan.placement.replicas]),
                slo=rt.Slo.latency(400_000), qps_max=plan.qps_max,
                gears=tuple(rt.Gear(rt.Cascade(g.cascade.stages, g.cascade.thresholds),
                                    dict(g.min_queue_length), dict(g.load_weights))
                            for g in plan.gears))
            from gearserve import synth as rsynth
            rprof = rsynth.make_profiles(4, (1.0, 4.0, 16.0, 64.0), base_runtime_us=1_000)
            rval = rsynth.make_validation(rprof, n_samples=2000, easy_fraction=0.8, seed=5)
            rsub = rt.WorkloadTrace(sub.arrivals[:20_000])
            t = time.perf_counter()
            m = reng.run(rplan, rsub, rval, rprof, config=reng.EngineConfig(seed=0))
            dt = time.perf_counter() - t
            out["cpu_baseline"]["reference_engine_run"] = {
                "routed_samples_per_s": sum(x.stages_executed for x in m.per_request) / dt,
                "requests_per_s": len(rsub) / dt, "cores": 1, "kind": "reference",
                "sample": "first 20k requests of group 0, baseline/_ref gearserve.engine.run"}
        except Exception as e:  # noqa: BLE001
            out["cpu_baseline"]["reference_engine_run"] = {"error": f"{type(e).__name__}: {e}"}
    # probes: SP1 burst-throughput probes (_burst_throughput), 1,024 per launch
    cands = []
    rng = np.random.default_rng(0)
    for _ in range(1024):
        k = int(rng.integers(1, 5))
        st = tuple(sorted(rng.choice(4, size=k, replace=False)))
        stages = tuple(f"m{i}" for i in st)
        thr = tuple(float(x) for x in np.round(rng.uniform(0.6, 0.9, k - 1), 3))
        cands.append(Cascade(stages, thr))
    pjobs = []
    for c in cands:
        w = {m: {r.replica_id: 1.0 for r in plan.placement.replicas_of(m)} for m in c.stages}
        q = {r.replica_id: 1 for m in c.stages for r in plan.placement.replicas_of(m)}
        pplan = GearPlan(placement=plan.placement, slo=None, qps_max=1.0, gears=(Gear(c, q, w),))
        serial = sum(prof[m].runtime_table[1] for m in c.stages)
        pjobs.append(replay.Job(replay.DevicePlan(pplan, prof, val), np.zeros(256, np.int64),
                                256 * serial * 2 + 1_000_000,
                                replay.EngineConfig(seed=0, enable_ticks=False)))
    pprep = replay.Prepared(pjobs)
    pprep.run()
    torch.cuda.synchronize()
    a_ev.record()
    pprep.run()  # one launch: 1,024 probes
    b_ev.record()
    torch.cuda.synchronize()
    pms = a_ev.elapsed_time(b_ev)
    pres = pprep.results()
    thr_probe = [r.completed / (int(r.records["completion_us"].max()) / 1e6) for r in pres[:4]]
    t = time.perf_counter()
    for c in cands[:64]:
        w = {m: {r.replica_id: 1.0 for r in plan.placement.replicas_of(m)} for m in c.stages}
        q = {r.replica_id: 1 for m in c.stages for r in plan.placement.replicas_of(m)}
        pplan = GearPlan(placement=plan.placement, slo=None, qps_max=1.0, gears=(Gear(c, q, w),))
        serial = sum(prof[m].runtime_table[1] for m in c.stages)
        oracle.engine_run(pplan, WorkloadTrace(np.zeros(256, np.int64),
                                               duration_us=256 * serial * 2 + 1_000_000),
                          cert, corr, runtime, [8] * 4, {m: j for j, m in enumerate(ids)},
                          seed=0, enable_ticks=False)
    probe_cpu = 64 / (time.perf_counter() - t)
    out["online_router"] = _guarded(online_router_bench, plan, prof, cert, corr)
    out["probes"] = {"probes": len(pjobs), "ms": pms, "probes_per_s": len(pjobs) / (pms * 1e-3),
                     "requests_per_probe": 256, "launches": 1,
                     "first_throughputs_qps": thr_probe,
                     "cpu_baseline": {"value": probe_cpu, "unit": "probes/s", "cores": 1,
                                      "kind": "port",
                                      "sample": "64 of the probes, oracle.engine_run, one core"}}
    del pprep
    return out


def cpu_baseline(cert, corr, grids, cost1, args):
    """Oracle port of _evaluate_numba on a bounded config sample, all threads."""
    from oracle import oracle
    threads = os.cpu_count() or 1
    sm, thr, ns = oracle.grid_configs(grids)
    rng = np.random.default_rng(2)
    batch = threads * 8
    pick = np.sort(rng.choice(sm.shape[0], size=batch, replace=False))
    oracle.evaluate_encoded(cert, corr, sm[pick[:threads]], thr[pick[:threads]],
                            ns[pick[:threads]], cost1, n_threads=threads)  # warm
    n, dt = 0, 0.0
    while dt < args.cpu_seconds:  # bounded sample: batches until the time budget is used
        pick = np.sort(rng.choice(sm.shape[0], size=batch, replace=False))
        t = time.perf_counter()
        oracle.evaluate_encoded(cert, corr, sm[pick], thr[pick], ns[pick], cost1,
                                n_threads=threads)
        dt += time.perf_counter() - t
        n += batch
    return {"value": n / dt, "unit": "config-evals/s", "cores": threads, "kind": "port",
            "sample": f"{n} configs sampled uniformly from the {sm.shape[0]} of cfg2, all 1M "
                      f"records each ({dt:.1f} s, oracle/oracle_eval.c, {threads} threads)"}


# ---------------------------------------------------------- reference -----
def run_reference(args, world, rank):
    if rank != 0:
        return
    from oracle import oracle
    _, cert, corr, grids, cost1 = workload(seed=0, device_grids=False)
    threads = os.cpu_count() or 1
    sm, thr, ns = oracle.grid_configs(grids)
    rng = np.random.default_rng(3)
    per_step = max(threads, 16) * 8  # 8 configs per thread: thread start-up amortised
    for _ in range(args.warmup):
        p = rng.choice(sm.shape[0], size=per_step, replace=False)
        oracle.evaluate_encoded(cert, corr, sm[p], thr[p], ns[p], cost1, n_threads=threads)
    t = time.perf_counter()
    for _ in range(args.steps):
        p = rng.choice(sm.shape[0], size=per_step, replace=False)
        oracle.evaluate_encoded(cert, corr, sm[p], thr[p], ns[p], cost1, n_threads=threads)
    dt = time.perf_counter() - t
    value = args.steps * per_step / dt
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "config-evals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "n_records": N_REC, "n_models": N_MODELS,
                   "grid_levels": LEVELS},
        "cpu_baseline": {"value": value, "unit": "config-evals/s", "cores": threads,
                         "kind": "port",
                         "sample": f"{per_step} random configs per step x all 1M records "
                                   f"(oracle/oracle_eval.c restating kernels._evaluate_numba)"},
        "e2e": {"value": value, "unit": "config-evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--skip-stage", action="store_true", help="skip the stage-step leg")
    ap.add_argument("--skip-ingest", action="store_true", help="skip the ingest leg")
    ap.add_argument("--skip-config4", action="store_true", help="skip the 5-stage (cfg4b) leg")
    ap.add_argument("--skip-config1", action="store_true", help="skip the 3-model cfg1 leg")
    ap.add_argument("--skip-list", action="store_true", help="skip the list-path legs")
    ap.add_argument("--skip-config3", action="store_true", help="skip the cfg3 cascade leg")
    ap.add_argument("--skip-config5", action="store_true", help="skip the cfg5 replay leg")
    ap.add_argument("--skip-config4a", action="store_true", help="skip the cfg4a front leg")
    ap.add_argument("--skip-head", action="store_true", help="skip the tensor-core head leg")
    ap.add_argument("--flush", choices=["write", "clean", "none"], default="write",
                    help="L2 eviction between timed steps (see flush_l2)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="CPU time budget of the cpu_baseline sample")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args, int(os.environ.get("WORLD_SIZE", "1")),
                      int(os.environ.get("RANK", "0")))
        return
    world, rank, local = init_dist()
    run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
