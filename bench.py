#!/usr/bin/env python
"""Benchmark of the augsched hot path on B200 (one JSON line on rank 0).

Workload (default "cfg5"): BASELINE.json config 5 per GPU — 65,536 simulated
serving instances = 4,096 synthetic W2 traces of 5,000 tool-augmented requests
(rates cycling 2/3/4/5 req/s) x 16 parameter points (4 target_max x 4 alpha),
7B cost-model preset.  One bench step = every instance advances through the
next `--window` simulated iterations (all of §8(a): intake, token limit,
scoring, ordering, admission, memory resolution, engine advance, metrics),
inside one persistent kernel launch.  Metric: scheduling decisions/s (sum of
queue sizes over busy steps, R27) with sim instance-steps/s beside it.

Multi-GPU (torchrun): weak scaling — each rank simulates its own 65,536
instances (trace ids offset by rank), no data-path collective; the per-rank
result records are all-gathered over NCCL at the end (north star).

--impl reference: the CPU oracle (oracle/) timed on this box's host cores on a
bounded sample of the same workload (rank 0 only).
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

import tracegen  # noqa: E402

METRIC = "scheduling decisions/s"
UNIT = "decisions/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="augsched", choices=["augsched", "reference"])
    ap.add_argument("--workload", default="cfg5", choices=["cfg5", "cfg3"])
    ap.add_argument("--instances", type=int, default=65536, help="instances per GPU (cfg5)")
    ap.add_argument("--window", type=int, default=1500, help="simulated iterations per bench step")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0, help="oracle sample size (instances)")
    ap.add_argument("--no-step", action="store_true", help="skip the cfg4 1M-queue step measurement")
    ap.add_argument("--step-n", type=int, default=1_000_000)
    return ap.parse_args()


# ----------------------------------------------------------------------------- workload
def workload_name(args):
    if args.workload == "cfg5":
        n_inst = args.instances
        return (f"cfg5: {n_inst} instances/GPU = {max(1, n_inst // 16)} W2 traces x 5000 requests (2-5 req/s, "
                f"math/QA/web/chatbot tool mix) x 16 params (target_max 250-1000 x alpha 0-1000M), 7B preset")
    return "cfg3: 4096 instances (64 target_max x 64 TTFT SLO) x 2000 requests @4 req/s, 7B preset"


def workload(args, rank):
    """Synthetic traces + per-instance parameters of this rank's shard."""
    if args.workload == "cfg5":
        n_inst = args.instances
        n_tr = max(1, n_inst // 16)
        # weak scaling: rank r owns trace ids [r*n_tr, (r+1)*n_tr) of the global set
        parts = [tracegen.gen_trace_arrays(5000, [2.0, 3.0, 4.0, 5.0][(rank * n_tr + i) % 4],
                                           5000, rank * n_tr + i) for i in range(n_tr)]
        req_off = np.arange(n_tr + 1, dtype=np.int64) * 5000
        cat = [np.concatenate([p[j] for p in parts]) for j in range(8)]
        tr = tracegen._finish(req_off, *cat)
        ip = tracegen.cfg5_params(n_inst)
        tid = (np.arange(n_inst) // 16).astype(np.uint32)
        return tr, ip, tid, 5000, workload_name(args)
    tr = tracegen.gen_traces(1, 2000, [4.0], seed=3)
    ip = tracegen.cfg3_params()
    tid = np.zeros(4096, np.uint32)
    return tr, ip, tid, 2000, workload_name(args)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu, self.rows, self.stop_ev = gpu, [], threading.Event()

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop_ev.wait(0.2)

    def __enter__(self):
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop_ev.set()
        self.th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------------------- oracle timing
def cpu_baseline(args, tr, ip, tid, iters, sample=None):
    """The oracle as it stands on a bounded sample: instances every `stride`,
    simulated for the same number of iterations as the GPU's timed region."""
    import oracle
    n = len(tid)
    k = sample or max(8, min(512, n // 128))
    idx = np.linspace(0, n - 1, k).astype(np.int64)
    sub = {kk: v[idx] for kk, v in ip.items()}
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    res = oracle.simulate(tracegen.PRESET_7B, sub, tr, tid[idx], max_iters=iters, threads=cores)
    dt = time.perf_counter() - t0
    dec = int(res["f"][:, oracle.FIELDS.index("decisions")].sum())
    steps = int(res["f"][:, oracle.FIELDS.index("busy_steps")].sum())
    return {"value": dec / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{k} of {n} instances (evenly spaced), iterations [0, {iters}), {dt:.1f} s wall",
            "instance_steps_per_s": steps / dt, "seconds": dt}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    tr, ip, tid, ma, name = workload(args, 0)
    iters = args.window * (args.warmup + args.steps)
    # each step: the oracle on a bounded sample of the same workload
    vals, secs = [], []
    for s in range(args.warmup + args.steps):
        cb = cpu_baseline(args, tr, ip, tid, args.window * (s + 1),
                          sample=args.cpu_sample or max(8, os.cpu_count() or 1))
        if s >= args.warmup:
            vals.append(cb["value"])
            secs.append(cb["seconds"])
    v = float(np.median(vals))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.median(secs)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": name, "window_iters": args.window},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
                             "sample": cb["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- cfg4 step
def step_bench(args, dev, stream, peak, prefix=False, n_override=None):
    """Config 4: one scheduling step over one 1,000,000-request queue, K
    consecutive steps, each timed with CUDA events after an L2 flush (the
    working set, ~60 MB, fits in L2).  prefix=False: augsched_step (scores,
    full stable order, admission, grant accounting); prefix=True:
    augsched_step_prefix (the same decisions, order produced for the
    admitted prefix only)."""
    import torch
    import paper_2512_04013_b200 as aug
    n = n_override or args.step_n
    rec = tracegen.cfg4_records(n)
    s = aug.Scheduler(tracegen.PRESET_CFG4, tracegen.inst_params(1), 1, n, device=dev, stream=stream)
    s.enqueue(0, rec)
    flush = torch.empty(512 * 2**20, dtype=torch.uint8, device=f"cuda:{dev}")
    t = 65536
    for _ in range(args.warmup):
        s.step(t, prefix=prefix); t += 1
    torch.cuda.synchronize()
    l0 = s.launches
    cold, warm = [], []
    for _ in range(args.steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream); s.step(t, prefix=prefix); b.record(stream); t += 1
        torch.cuda.synchronize()
        cold.append(a.elapsed_time(b))
    for _ in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream); s.step(t, prefix=prefix); b.record(stream); t += 1
        torch.cuda.synchronize()
        warm.append(a.elapsed_time(b))
    launches = (s.launches - l0) // (2 * args.steps)
    s.close()
    ms = float(np.median(cold))
    ach = 32.0 * n / (ms / 1e3) / 1e9
    what = ("augsched_step_prefix: one cooperative kernel, one launch (streaming pass: Eq.26 key of every "
            "slot, words at or below the previous step's anchor kept as candidates; one CTA sorts them and "
            "admits/resolves/applies; histogram fallback when the anchor fails)"
            if prefix else "augsched_step: keys + 4 LSD sort passes + admit/resolve/apply")
    traffic = None
    if prefix:   # ncu DRAM bytes per steady launch of the same command (profiles/step_prefix_traffic.json)
        try:
            tj = json.load(open(os.path.join(ROOT, "profiles", "step_prefix_traffic.json")))
            traffic = tj["sizes"].get(str(n), {}).get("dram_bytes_per_launch_mean")
        except (OSError, ValueError, KeyError):
            traffic = None
    return {"workload": f"cfg4: one queue of {n} requests (512 running, 512 swapped, rest waiting "
                        "80% Stage I / 20% Stage II), " + ("admitted prefix" if prefix else "full stable order") +
                        " + admission per step",
            "value": n / (ms / 1e3), "unit": UNIT, "ms_per_step_cold_l2": ms,
            "ms_per_step_warm_l2": float(np.median(warm)), "launches_per_step": launches,
            "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(ach / peak, 4), "traffic": traffic,
                         "note": what + "; 32 B/decision, whole step, L2 flushed before each step"}}


def step_multi_bench(args, dev, stream, peak, n_inst=4096, ma=2048):
    """The batched scheduler: one augsched_step / augsched_step_prefix call
    for n_inst serving instances of `ma` slots each (cfg4-shaped queues),
    L2 flushed before each step."""
    import torch
    import paper_2512_04013_b200 as aug
    rec = tracegen.cfg4_records(ma, n_running=16, n_swapped=16, n_paused=4)
    flush = torch.empty(512 * 2**20, dtype=torch.uint8, device=f"cuda:{dev}")
    res = {"workload": f"{n_inst} instances x {ma} slots (cfg4-shaped queues), one step call for all"}
    for prefix in (False, True):
        s = aug.Scheduler(tracegen.PRESET_CFG4, tracegen.inst_params(n_inst), n_inst, ma, device=dev, stream=stream)
        for i in range(n_inst):
            s.enqueue(i, rec)
        t = 65536
        for _ in range(args.warmup):
            s.step(t, prefix=prefix); t += 1
        ms = []
        for _ in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream); s.step(t, prefix=prefix); b.record(stream); t += 1
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        s.close()
        m = float(np.median(ms))
        n = n_inst * ma
        res["prefix" if prefix else "full_order"] = {
            "value": n / (m / 1e3), "unit": UNIT, "ms_per_step_cold_l2": m,
            "roofline_frac": round(32.0 * n / (m / 1e3) / 1e9 / peak, 4)}
    return res


# ----------------------------------------------------------------------------- GPU arm
def run_gpu(args):
    import torch
    import paper_2512_04013_b200 as aug
    from paper_2512_04013_b200 import _build

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    # AUGSCHED_BENCH_BACKEND=gloo: a test mode that runs N ranks on however
    # many GPUs the box has (device = local_rank mod count), collectives on
    # host copies; the default is one rank per GPU over NCCL.
    backend = os.environ.get("AUGSCHED_BENCH_BACKEND", "nccl")
    if world > 1:
        import torch.distributed as dist
        local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)

    def allreduce_(t, op):
        if backend == "nccl":
            dist.all_reduce(t, op=op)
            return t
        h = t.cpu()
        dist.all_reduce(h, op=op)
        t.copy_(h)
        return t
    if rank == 0:
        _build.build()
    if dist:
        dist.barrier()
    dev = torch.cuda.current_device()
    tr, ip, tid, ma, name = workload(args, rank)
    n_inst = len(tid)
    stream = torch.cuda.current_stream()
    s = aug.Scheduler(tracegen.PRESET_7B, ip, n_inst, ma, device=dev, stream=stream)
    dtr = aug.DeviceTraces(tr, device=f"cuda:{dev}")
    tid_d = torch.from_numpy(tid.astype(np.int32)).to(f"cuda:{dev}")
    out = torch.empty(n_inst * aug.RESULT_DTYPE.itemsize, dtype=torch.uint8, device=f"cuda:{dev}")
    W = args.window

    def field(res, name_):
        return int(res["f"][:, aug.RESULT_FIELDS.index(name_)].sum())

    # warm-up windows
    t_end = 0
    for _ in range(args.warmup):
        t_end += W
        s.simulate(dtr, tid_d, t_end, out=out, resume=t_end > W)
    torch.cuda.synchronize()
    before = aug.results_to_numpy(out)
    l0 = s.launches
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        for k in range(args.steps):
            t_end += W
            evs[k][0].record(stream)
            s.simulate(dtr, tid_d, t_end, out=out, resume=True)
            evs[k][1].record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches = s.launches - l0
    ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = float(sum(ms))
    after = aug.results_to_numpy(out)
    dec = field(after, "decisions") - field(before, "decisions")
    isteps = field(after, "busy_steps") - field(before, "busy_steps")
    tm = torch.tensor([total_ms, dec, isteps], dtype=torch.float64, device=f"cuda:{dev}")
    if dist:
        mx = tm.clone()
        allreduce_(mx, dist.ReduceOp.MAX)
        tot = tm.clone()
        allreduce_(tot, dist.ReduceOp.SUM)
        tm = torch.stack([mx[0], tot[1], tot[2]])
        # final NCCL all-gather of the per-instance result records (north star)
        from paper_2512_04013_b200 import dist as adist
        g0 = time.perf_counter()
        gathered = adist.all_gather_records(out, world)
        torch.cuda.synchronize()
        gather_ms = 1e3 * (time.perf_counter() - g0)
        assert gathered.numel() == world * out.numel()
    else:
        gather_ms = 0.0
    total_ms, dec_all, isteps_all = float(tm[0]), float(tm[1]), float(tm[2])
    value = dec_all / (total_ms / 1e3)

    # ---- roofline of the dominant (only) kernel: §8(d) 32 B per decision
    import json as _j
    peaks = {}
    try:
        peaks = _j.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        peak, peak_src = float(peaks["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        peak, peak_src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
    per_launch_bytes = 32.0 * dec / max(1, args.steps)
    achieved = per_launch_bytes / (total_ms / args.steps / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": None,
            "kernel": "sim_kernel (persistent; 16 one-warp instances per CTA advancing in step)", "peak_source": peak_src,
            "algorithmic_bytes_per_decision": 32}
    # DRAM bytes per launch of the same kernel on the same workload, from one
    # ncu capture of bench.py's timed launches (tools/traffic.py)
    prof = os.path.join(ROOT, "profiles", "sim_kernel_traffic.json")
    if os.path.exists(prof):
        try:
            pj = _j.load(open(prof))
            if pj.get("workload") == name and pj.get("window_iters", W) == W:
                roof["traffic"] = pj["dram_bytes_per_launch_mean"]
                roof["traffic_source"] = "profiles/sim_kernel_traffic.json (ncu, same workload)"
        except Exception:
            pass

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": name, "window_iters": W, "instances_per_gpu": n_inst,
                       "l2": "inputs larger than L2 (per-GPU state %.1f GB)" % (
                           n_inst * ma * 100 / 1e9)},
            "instance_steps_per_s": isteps_all / (total_ms / 1e3),
            "gpu_launches": launches, "roofline": roof, "allgather_ms": gather_ms}
    line["clocks"] = clk.summary()

    # ---- end to end through the C ABI with host buffers (pinned), rank-local
    if not args.no_e2e:
        s2 = aug.Scheduler(tracegen.PRESET_7B, ip, n_inst, ma, device=dev, stream=stream)
        pinned = aug.PinnedTraces(tr)
        t_e = 0
        for _ in range(args.warmup):
            t_e += W
            s2.simulate_host(pinned, tid, t_e, resume=t_e > W)
        before_e = s2.simulate_host(pinned, tid, t_e, resume=True)  # no-op window: snapshot
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            t_e += W
            res_e = s2.simulate_host(pinned, tid, t_e, resume=True)
        ev1.record(stream)
        torch.cuda.synchronize()
        e_ms = ev0.elapsed_time(ev1)
        dec_e = field(res_e, "decisions") - field(before_e, "decisions")
        et = torch.tensor([e_ms, dec_e], dtype=torch.float64, device=f"cuda:{dev}")
        if dist:
            m = et.clone()
            allreduce_(m, dist.ReduceOp.MAX)
            tot = et.clone()
            allreduce_(tot, dist.ReduceOp.SUM)
            et = torch.stack([m[0], tot[1]])
        line["e2e"] = {"value": float(et[1]) / (float(et[0]) / 1e3), "unit": UNIT,
                       "h2d_bytes_per_step": pinned.nbytes + 4 * n_inst,
                       "d2h_bytes_per_step": n_inst * aug.RESULT_DTYPE.itemsize}
        s2.close()
    if rank == 0 and not args.no_step:
        line["step_1m"] = step_bench(args, dev, stream, peak)
        line["step_1m_prefix"] = step_bench(args, dev, stream, peak, prefix=True)
        # size sweep of the prefix step: queues beyond L2 show the HBM-bound regime
        sweep = {}
        for n_sw in (4_194_304, 16_000_000):
            r_sw = step_bench(args, dev, stream, peak, prefix=True, n_override=n_sw)
            sweep[str(n_sw)] = {"value": r_sw["value"], "ms_per_step_cold_l2": r_sw["ms_per_step_cold_l2"],
                                "roofline_frac": r_sw["roofline"]["frac"],
                                "achieved_gbs": r_sw["roofline"]["achieved"]}
        line["step_1m_prefix"]["size_sweep"] = sweep
        line["step_multi"] = step_multi_bench(args, dev, stream, peak)
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args, tr, ip, tid, W * (args.warmup + args.steps),
                                            sample=args.cpu_sample or None)
    s.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    run_gpu(args)


if __name__ == "__main__":
    main()
