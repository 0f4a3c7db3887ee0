#!/usr/bin/env python
"""bench.py — throughput of the B200-native CRM SPH particle update (one JSON line on rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config bed32M] [--impl ours|reference]

A "step" is one full pass of the hot path (SURVEY.md §8(a) A1–A8: bin, sort, reorder, neighbour
lists, BCE extrapolation x2, fused rates + RK2 epilogues + return map) over the whole workload.
Default workload: BASELINE.json configs[4], the synthetic 32M-particle granular bed (1024 x 512 x 64
fluid at d0 = 5 mm, h = 1.3 d0 = 6.5 mm, 2.22M wall markers), the largest configuration that fits one
GPU.  The state (~2 GB) is larger than L2, so no L2 flush is needed between timed steps.

Timing: W untimed warm-up steps, then K steps bracketed by barrier + cudaStreamSynchronize, timed with
CUDA events on the library's stream; max over ranks.  Per-kernel device times come from the library's
own event pairs (crm_profile_*) over the same timed region.  `e2e` re-measures the metric through the
public C-ABI with pinned host buffers: every step uploads the fluid state (crm_set_state), steps, and
reads it back (crm_get_state).  `cpu_baseline` times the fp64 oracle (oracle/) on a bounded sample of
the same workload on the host cores (rank 0, N = 1 only).  `--impl reference` times that oracle as the
reference arm.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

METRIC = "SPH particle-updates/sec and ms/step at 1/2/4/8 B200; % of HBM roofline"
UNIT = "particle-updates/s"

# algorithmic work: FP32 flops per directed pair of the rates loop, per
# neighbour-search candidate, per marker-fluid pair; epilogue flops per fluid particle
FLOPS_PER_PAIR = 84
FLOPS_PER_CANDIDATE = 8
FLOPS_PER_BCE_PAIR = 30
FLOPS_EPILOGUE = {"k_rates_A": 110, "k_rates_B": 170}
# FP32-pipe issue slots per unit of algorithmic work (~63 per directed pair of the
# rates loop, ~7 per neighbour-search candidate) against 148 SM x 128 lanes x f_SM slots/s (D5)
SLOTS_PER_PAIR = 63
SLOTS_PER_CANDIDATE = 7
# algorithmic HBM bytes per fluid particle-update and per BCE marker
BYTES_PER_FLUID_UPDATE = 404
BYTES_PER_BCE_UPDATE = 72
# (the 56-B fp32 state of D4; the 16-B position compensation term L is this design's overhead)
# bounded oracle sample of the bed workload (~1M fluid; ~1 s per oracle step on a 16-core host)
SAMPLE_BED = (128, 128, 64)
# the 1-thread oracle sample (~262k fluid, a few seconds per step on one core)
SAMPLE_BED_1T = (64, 64, 64)
# per-kernel bytes per particle of the HBM-bound kernels (reorder moves the 72-B state incl. L)
KERNEL_BYTES = {"k_bin": 16 + 4 + 8 + 4, "k_scatter": 12 + 8, "k_reorder": 72 + 72 + 24 + 8}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm_gbs=d["hbm_gbs"], sm_max_mhz=d.get("sm_max_mhz", 1965.0), source="measured")
    return dict(hbm_gbs=6650.0, sm_max_mhz=1965.0, source="fallback")


def fp32_peak_tflops(mhz):
    # 148 SMs x 128 FP32 lanes x 2 flops (FFMA) per clock (B200_PROFILING.md unit counts)
    return 148 * 128 * 2 * mhz * 1e6 / 1e12


def scenario(name: str):
    if name == "bed32M":
        return workloads.bed()
    if name.startswith("bed"):
        nx, ny, nz = (int(t) for t in name[3:].split("x"))
        return workloads.bed(n=(nx, ny, nz))
    if name == "block8k":
        return workloads.block_settle()
    if name == "cone1M":
        return workloads.cone_bed()
    if name == "mgru3":
        return workloads.mgru3_bin()
    if name == "crater":
        return workloads.cratering()
    raise SystemExit(f"unknown config {name}")


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [t.strip() for t in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[3:7]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for _, _, r in rows for k in range(4) if r[k].lower() == "active"})
        return {"sm_mhz": float(np.median([r[0] for r in rows])), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ oracle timing
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_rate(name: str, steps: int, one_thread: bool = True):
    """Time the fp64 oracle (as it stands) on a bounded sample of the workload on the host's cores,
    and on one core (a smaller sample of the same recipe)."""
    import oracle
    oracle.build()
    if name.startswith("bed"):
        sample = workloads.bed(n=SAMPLE_BED)
        desc = (f"{SAMPLE_BED[0]}x{SAMPLE_BED[1]}x{SAMPLE_BED[2]}-fluid sub-bed of the bed recipe "
                "(same d0, h, material, dt)")
    else:
        sample = scenario(name)
        desc = f"full {name} workload"
    s = oracle.load_scenario(sample)
    t0 = time.perf_counter()
    s.step(sample.dt, steps)
    t = time.perf_counter() - t0
    out = dict(value=sample.n_fluid * steps / t, unit=UNIT, cores=oracle.num_threads(), kind="oracle",
               cpu_model=cpu_model(),
               sample=f"{desc}; {steps} step(s) in {t:.2f} s; {sample.n_fluid + sample.n_bce} particles")
    if one_thread:
        nthr = oracle.num_threads()
        s1 = workloads.bed(n=SAMPLE_BED_1T) if name.startswith("bed") else sample
        o1 = oracle.load_scenario(s1)
        oracle.set_num_threads(1)
        try:
            t0 = time.perf_counter()
            o1.step(s1.dt, 1)
            t1 = time.perf_counter() - t0
        finally:
            oracle.set_num_threads(nthr)
        out["one_thread"] = {"value": s1.n_fluid / t1, "unit": UNIT, "cores": 1,
                             "sample": f"{s1.n_fluid} fluid + {s1.n_bce} BCE; 1 step in {t1:.2f} s"}
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        # torchrun pins OMP_NUM_THREADS=1 per rank; rank 0 runs alone here, so the oracle gets the
        # host's cores as at N = 1 (read by libgomp when liboracle loads, below)
        os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    cb = oracle_rate(args.config, max(1, args.steps + args.warmup) if args.config == "block8k" else 1, one_thread=False)
    # warm-up + timed steps of the oracle itself on the sample (bounded: one sample step per bench step)
    import oracle
    sample = workloads.bed(n=SAMPLE_BED) if args.config.startswith("bed") else scenario(args.config)
    s = oracle.load_scenario(sample)
    s.step(sample.dt, args.warmup)
    t0 = time.perf_counter()
    s.step(sample.dt, args.steps)
    t = time.perf_counter() - t0
    val = sample.n_fluid * args.steps / t
    cb = dict(cb, value=val, sample=cb["sample"].split(";")[0] + f"; {args.steps} timed steps in {t:.2f} s")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": args.config, "sample_fluid": sample.n_fluid},
            "cpu_baseline": cb,
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def ps_freq_of(sc) -> int:
    return int(sc.params.get("ps_freq", 1) or 1)


def active_measure(crm, torch, local, warmup, steps):
    """ms/step of the MGRU3 wheel bin with and without active domains (same input, same steps)."""
    out = {"workload": "mgru3_wheel", "active_box_m": [0.6, 0.6, 0.8], "steps": steps}
    for on in (False, True):
        sc = workloads.mgru3_wheel(active=on)
        g = crm.load_scenario(sc, device=local)
        st = torch.cuda.ExternalStream(g.stream(), device=local)
        g.step(sc.dt, warmup)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.step(sc.dt, steps)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        key = "on" if on else "off"
        out[f"ms_per_step_{key}"] = ms
        if on:
            s = g.active_stats()
            out.update(n_total=g.count(), n_active=s["active"], n_extended=s["extended"],
                       n_inactive=s["inactive"], capacity=s["capacity"])
        else:
            out["n_fluid"] = sc.n_fluid
        g.close()
    out["speedup"] = out["ms_per_step_off"] / out["ms_per_step_on"]
    out["note"] = ("Alg. 3 (P:876-947): UpdateActivity + compaction + ManageArrayMemory each rebuild, "
                   "ps_freq = 1; paper Table tab:active_domains_performance: MGRU3 wheel 2.93x, "
                   "RASSOR drum 2.11x (whole co-simulation RTF, its hardware)")
    return out


def cone_measure(crm, torch, local, warmup, steps_total=1500, every=150):
    """The cone penetration test on the full C3 bed: 60 deg cone, fall from H = L;
    ms/step and the depth-vs-time curve of the tip below the initial surface."""
    sc = workloads.cone_drop(H_over_L=1.0)
    g = crm.load_scenario(sc, device=local)
    st = torch.cuda.ExternalStream(g.stream(), device=local)
    surface = sc.meta["n"][2] * sc.params["d0"]
    curve, ms = [], 0.0
    for _ in range(steps_total // every):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.step(sc.dt, every)
        e1.record(st)
        torch.cuda.synchronize()
        ms += e0.elapsed_time(e1)
        tip = g.get_body(1)["pos"][2] - 0.75 * sc.meta["cone_L"]
        curve.append([round((len(curve) + 1) * every * sc.dt, 6), round(surface - tip, 6)])
    g.close()
    n = (steps_total // every) * every
    return {"workload": sc.name, "n_fluid": sc.n_fluid, "n_bce": sc.n_bce, "steps": n,
            "ms_per_step": ms / n, "value": sc.n_fluid / (ms / n * 1e-3), "unit": UNIT,
            "depth_vs_time_s_m": curve,
            "note": "free 60 deg / 19.8 mm steel cone (reading A32) entering with sqrt(2 g L); the paper "
                    "compares this curve with experiments (P:100), which are not reproduced here"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="bed32M")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--repeats", type=int, default=5, help="timed K-step regions; the median is reported (SURVEY D6: median of 5)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-next", action="store_true", help="skip the ps_freq = 10 (Alg. 2) measurement")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    assert args.warmup >= 3, "timing rules: at least 3 warm-up steps"

    import torch
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    nccl_log = None
    if world > 1:
        # NCCL's INFO lines (communicator size, transports, NVLS) go to a per-rank file: rank 0 reports
        # its communicator lines in the JSON so the scaling run can be checked against the rank count
        nccl_log = f"/tmp/crm_nccl.{rank}.{os.getpid()}.log"
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_FILE", nccl_log)
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        dist = None
    torch.cuda.set_device(local)

    from paper_2507_05643_b200 import build as _b
    _b.build_library()
    from paper_2507_05643_b200 import crm

    sc = scenario(args.config)
    n_fluid, n_bce = sc.n_fluid, sc.n_bce
    # N > 1: slab decomposition along x with NCCL halo exchanges inside libcrm;
    # every rank passes the same global input and keeps its slab
    if world > 1:
        from paper_2507_05643_b200 import dist as cdist
        nid = cdist.bootstrap_nccl_id(rank)
        g = crm.load_scenario(sc, device=local, rank=rank, world=world, nccl_id=nid)
    else:
        g = crm.load_scenario(sc, device=local)
    stream = torch.cuda.ExternalStream(g.stream(), device=local)

    def barrier():
        if dist is not None:
            dist.barrier()

    # warm-up (the first step also builds the NCCL communicator)
    barrier()
    g.step(sc.dt, args.warmup)
    # directed fluid pairs of this rank (algorithmic work of the rates kernels)
    pairs_local = g.pair_count()
    pairs_fluid = pairs_local
    cand_local, cand_markers = g.candidate_count()   # Alg. 1 candidate tests (filter work)
    if dist is not None:
        t = torch.tensor([pairs_local], dtype=torch.int64, device=f"cuda:{local}")
        dist.all_reduce(t)
        pairs_fluid = int(t.item())

    # headline: K steps replayed from the library's CUDA graphs, CUDA events on its stream; the K-step
    # region is timed R times (barrier + synchronize around each) and the median is reported
    clk = ClockSampler(local)
    clk.start()
    reps = []
    launches = 0
    for _ in range(max(1, args.repeats)):
        barrier()
        torch.cuda.synchronize()
        n0 = g.launch_count()
        ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        g.step(sc.dt, args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
        launches = g.launch_count() - n0
        r = ev0.elapsed_time(ev1)
        if dist is not None:
            t = torch.tensor([r], device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            r = float(t.item())
        reps.append(r)
    clocks = clk.stop()
    ms = float(np.median(reps))
    # per-kernel device times: the same K steps again, launched kernel by kernel with an event
    # pair around every launch (crm_profile_*); not part of the headline
    g.profile(True)
    g.profile_reset()
    barrier()
    torch.cuda.synchronize()
    g.step(sc.dt, args.steps)
    torch.cuda.synchronize()
    prof = g.profile_read()
    g.profile(False)
    ms_step = ms / args.steps
    value = n_fluid / (ms_step * 1e-3)     # the whole job: every fluid particle, once per step

    pk = peaks()
    # dominant kernel and its roofline
    dom = max(prof.items(), key=lambda kv: kv[1][0])
    dname, (dms, dl) = dom
    per_launch_s = dms / dl * 1e-3
    if dname in ("k_rates_A", "k_rates_B", "k_filter"):
        n_own = g.count(crm.CRM_OWNED) if world > 1 else n_fluid
        if dname == "k_filter":   # Alg. 1: one B2 predicate per candidate (fluid and marker lists)
            flops = (cand_local + cand_markers) * FLOPS_PER_CANDIDATE
        else:
            flops = pairs_local * FLOPS_PER_PAIR + min(n_own, n_fluid) * FLOPS_EPILOGUE[dname]
        achieved = flops / per_launch_s / 1e12
        peak = fp32_peak_tflops(pk["sm_max_mhz"])
        roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "kernel": dname, "algorithmic_flops_per_launch": flops, "flops_per_pair": FLOPS_PER_PAIR,
                "pairs": pairs_local, "candidates": cand_local + cand_markers,
                "flops_per_candidate": FLOPS_PER_CANDIDATE,
                "share_of_step": dms / args.steps / ms_step,
                "fp32_issue_frac": ((cand_local + cand_markers) * SLOTS_PER_CANDIDATE if dname == "k_filter"
                                    else pairs_local * SLOTS_PER_PAIR) / per_launch_s
                                   / (148 * 128 * pk["sm_max_mhz"] * 1e6),
                "fp32_issue_note": "SURVEY D3/D5: 7 issue slots per candidate, 63 per directed pair, over "
                                   "148 x 128 lanes x sm_max_mhz",
                "peak_note": "148 SM x 128 FP32 lanes x 2 x sm_max_mhz (DESIGN.md §Roofline)"}
    else:
        nbytes = (n_fluid + n_bce) * KERNEL_BYTES.get(dname, 56)
        achieved = nbytes / per_launch_s / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "kernel": dname}
    roof["traffic"] = None
    prof_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof_path):
        tj = json.load(open(prof_path))
        tr = tj.get(args.config, {}).get(dname)
        if tr is not None:
            roof["traffic"] = tr
            roof["traffic_source"] = ("committed ncu --set full capture (profiles/ncu_traffic.json, "
                                      f"{tj.get('_source', 'see profiles/')}), not measured in this run")
    roof["peak_source"] = pk["source"]
    alg_bytes = n_fluid * BYTES_PER_FLUID_UPDATE + n_bce * BYTES_PER_BCE_UPDATE
    hbm = {"bytes_per_step": alg_bytes, "achieved_gbs": alg_bytes / (ms_step * 1e-3) / 1e9,
           "peak_gbs": pk["hbm_gbs"], "frac": alg_bytes / (ms_step * 1e-3) / 1e9 / pk["hbm_gbs"]}
    kernels = {k: {"ms_per_step": v[0] / args.steps, "launches": v[1]} for k, v in sorted(prof.items())}
    # whole step against the FP32 ALU roof: the step's algorithmic flops (both pair
    # stages, the Alg. 1 candidates, the epilogues) over the step time
    n_own_s = g.count(crm.CRM_OWNED) if world > 1 else n_fluid
    step_flops = (2 * pairs_local * FLOPS_PER_PAIR + (cand_local + cand_markers) * FLOPS_PER_CANDIDATE
                  + min(n_own_s, n_fluid) * (FLOPS_EPILOGUE["k_rates_A"] + FLOPS_EPILOGUE["k_rates_B"]))
    alu_step = {"flops_per_step": step_flops, "achieved_tflops": step_flops / (ms_step * 1e-3) / 1e12,
                "peak_tflops": fp32_peak_tflops(pk["sm_max_mhz"]),
                "frac": step_flops / (ms_step * 1e-3) / 1e12 / fp32_peak_tflops(pk["sm_max_mhz"]),
                "note": "per rank; 2 x pairs x 84 + candidates x 8 + epilogues 110 + 170 per fluid particle"}
    # the same ALU roofline for each of the three hot kernels (the line's `roofline` is the largest)
    n_own_k = g.count(crm.CRM_OWNED) if world > 1 else n_fluid
    for k in ("k_filter", "k_rates_A", "k_rates_B"):
        if k in prof and prof[k][1]:
            fl = ((cand_local + cand_markers) * FLOPS_PER_CANDIDATE if k == "k_filter"
                  else pairs_local * FLOPS_PER_PAIR + min(n_own_k, n_fluid) * FLOPS_EPILOGUE[k])
            tf = fl / (prof[k][0] / prof[k][1] * 1e-3) / 1e12
            kernels[k].update({"alu_tflops": tf, "alu_frac": tf / fp32_peak_tflops(pk["sm_max_mhz"])})
            slots = ((cand_local + cand_markers) * SLOTS_PER_CANDIDATE if k == "k_filter"
                     else pairs_local * SLOTS_PER_PAIR)
            kernels[k]["fp32_issue_frac"] = (slots / (prof[k][0] / prof[k][1] * 1e-3)
                                             / (148 * 128 * pk["sm_max_mhz"] * 1e6))

    # e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        n = n_fluid
        pin = lambda *shape: torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()  # noqa: E731
        pos, vel, rho, sig = pin(n, 3), pin(n, 3), pin(n), pin(n, 6)
        g.get_state(0, n, out=(pos, vel, rho, sig))
        ke = max(1, args.e2e_steps)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(ke):
            g.set_state(0, pos, vel, rho, sig)
            g.step(sc.dt, 1)
            g.get_state(0, n, out=(pos, vel, rho, sig))
        torch.cuda.synchronize()
        te = time.perf_counter() - t0
        if dist is not None:
            t = torch.tensor([te], device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        nbytes = n * 13 * 8
        e2e = {"value": n / (te / ke), "unit": UNIT, "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": nbytes, "steps": ke,
               "note": "per step: crm_set_state(all fluid, fp64 pinned) + crm_step(dt,1) + crm_get_state; host wall clock"}

    # the same workload with persistent neighbour lists (Alg. 2, ps_freq = 10);
    # a separate context, timed the same way (reported beside the ps_freq = 1 headline, not instead)
    nxt = None
    if not args.no_next:
        g.close()
        sc10 = scenario(args.config)
        sc10.params["ps_freq"] = 10
        if world > 1:
            g10 = crm.load_scenario(sc10, device=local, rank=rank, world=world, nccl_id=cdist.bootstrap_nccl_id(rank))
        else:
            g10 = crm.load_scenario(sc10, device=local)
        s10 = torch.cuda.ExternalStream(g10.stream(), device=local)
        barrier()
        g10.step(sc10.dt, args.warmup)
        barrier()
        torch.cuda.synchronize()
        k10 = 10 * max(1, args.steps // 10)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s10)
        g10.step(sc10.dt, k10)
        e1.record(s10)
        torch.cuda.synchronize()
        barrier()
        t10 = e0.elapsed_time(e1)
        if dist is not None:
            t = torch.tensor([t10], device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t10 = float(t.item())
        nxt = {"ps_freq": 10, "steps": k10, "ms_per_step": t10 / k10, "value": n_fluid / (t10 / k10 * 1e-3),
               "unit": UNIT, "speedup_vs_ps1": ms_step / (t10 / k10),
               "note": "Alg. 2 persistent lists (P:770-806): rebuild every 10 steps; paper: 1.28-1.36x (P:866)"}
        g10.close()

    # active domains (Alg. 3) on the MGRU3 wheel bin (1M particles, the
    # paper's 0.6 x 0.6 x 0.8 m active box around a prescribed rolling wheel), on vs off
    nxt_active = None
    nxt_cone = None
    if not args.no_next and world == 1 and rank == 0:
        nxt_active = active_measure(crm, torch, local, args.warmup, max(10, args.steps))
        nxt_cone = cone_measure(crm, torch, local, args.warmup)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_rate(args.config, 12)

    nccl_info = None
    if nccl_log and os.path.exists(nccl_log):
        keys = ("nRanks", "nranks", "Init COMPLETE", "NVLS", "Channel 00")
        nccl_info = [ln.strip()[:200] for ln in open(nccl_log, errors="replace") if any(k in ln for k in keys)][:8]
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
                "repeats_ms_per_step": [r / args.steps for r in reps],
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": args.config, "n_fluid": n_fluid, "n_bce": n_bce, "d0": sc.params["d0"],
                           "h": sc.params["h"], "dt": sc.dt, "pairs_fluid": pairs_fluid,
                           "particle_updates_incl_bce_per_s": (n_fluid + n_bce) / (ms_step * 1e-3),
                           "l2": "inputs larger than L2 (56 B x N state >> 126 MB), no flush",
                           "parallelism": f"x-slabs x{world}, NCCL ghost planes" if world > 1 else "single GPU"},
                "roofline": roof, "hbm_roofline": hbm, "alu_roofline_step": alu_step, "kernels": kernels, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clocks, "next_alg2": nxt, "next_active": nxt_active,
                "next_cone": nxt_cone, "nccl_info": nccl_info}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
