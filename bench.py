"""CoNet-Rx batched inference benchmark (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg2]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (BASELINE.json metric "CoNet-Rx inference slots/s and REs/s ... p50 per-slot latency",
quoted on configs[1] = cfg2): one step = featurize -> 3 ResNet subnetworks -> mul+BN fusion -> 1x1
LLR head over B=256 seeded synthetic slots per GPU (612 subcarriers x 14 symbols, 2 RX antennas,
16-QAM, TDL 12 taps / 300 ns / Jakes <= 200 Hz, SNR U[0,25] dB).  Slots are sharded across ranks
with no data-path collective (weak scaling: B per GPU is fixed).

  value   slots/s, inputs resident in HBM, device time (CUDA events on the launching stream), L2
          flushed (256 MiB write) between timed steps, max over ranks
  e2e     slots/s through the C-ABI host call cnrx_receive (pinned host y in, host LLRs out; H2D + D2H
          inside the timed region)
  roofline  dominant kernel: algorithmic FLOPs per launch (2 x MACs over all taps) /
          its average launch time from per-launch CUDA events over a second pass of the same K timed
          steps (events between launches cancel programmatic dependent launch, so the `value` pass
          runs without them), against the measured sustained bf16 peak in MEASURED_PEAKS.json
  cpu_baseline  the reference's own Network<float>::forward (oracle/_ref, compiled in place from
          /root/reference) + the restated featurizer, all host threads, bounded sample
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

METRIC = "CoNet-Rx inference slots/s and REs/s at 1/2/4/8 B200; p50 per-slot latency"
REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return d.get("bf16_tflops_sustained", 1383.6), d.get("hbm_gbs", 6536.0), "measured (MEASURED_PEAKS.json)"
    return 1400.0, 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms while the timed region runs."""

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,power.draw,power.limit",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, pw, pl = [], [], set(), [], []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                bits = int(parts[2], 16)
            except ValueError:
                continue
            try:
                pw.append(float(parts[3]))
                pl.append(float(parts[4]))
            except (ValueError, IndexError):
                pass
            for b, name in REASON_BITS.items():
                if bits & b and name != "gpu_idle":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        out = {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
               "samples": len(sm)}
        if pw:
            out["power_w"] = float(np.median(pw))
            out["power_limit_w"] = float(max(pl)) if pl else None
        return out


def cpu_baseline(cfg, g, batch, sample_slots=None, reps=1):
    """The reference's own forward (oracle/_ref) + the restated featurizer on this host's cores."""
    cores = os.cpu_count() or 1
    os.environ.setdefault("CONETRX_THREADS", str(cores))
    os.environ.pop("CONETRX_DETERMINISTIC", None)
    import oracle
    n = sample_slots or min(batch.y.shape[0], 2 * cores)
    y = batch.y[:n]
    if oracle.ref_available():
        net = oracle.RefNet.from_graph(g)
        kind, threads = "reference", int(oracle.ref().ref_threads())
        fwd = lambda x: net.forward(x)
    else:
        kind, threads = "port", 1
        fwd = lambda x: oracle.forward(g, x)
    t0 = time.perf_counter()
    for _ in range(reps):
        feat = oracle.featurize(y, batch.pilots, batch.pilot_mask)
        fwd(feat)
    dt = time.perf_counter() - t0
    slots_s = n * reps / dt
    return {"value": slots_s, "unit": "slots/s", "cores": threads, "kind": kind,
            "sample": f"{n} {cfg.name} slots x {reps} rep(s): restated featurize + reference Network<float>::forward"
                      f" (eval), CONETRX_THREADS={os.environ.get('CONETRX_THREADS')}, {dt:.1f} s"}


def run_reference(args, cfg, g):
    rank, local, world = dist_env()
    if rank != 0:
        return
    from paper_2510_12739_b200 import slots
    cores = os.cpu_count() or 1
    per_step = max(1, min(cfg.batch, cores))
    batch = slots.generate(cfg.link, per_step, seed=1000)
    os.environ.setdefault("CONETRX_THREADS", str(cores))
    import oracle
    if oracle.ref_available():
        net = oracle.RefNet.from_graph(g)
        kind, threads = "reference", int(oracle.ref().ref_threads())
        fwd = lambda x: net.forward(x)
    else:
        kind, threads = "port", 1
        fwd = lambda x: oracle.forward(g, x)

    def step():
        fwd(oracle.featurize(batch.y, batch.pilots, batch.pilot_mask))

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    v = per_step * args.steps / dt
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "slots/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "res_per_s": v * cfg.link.T * cfg.link.F,
            "config": {"workload": f"{cfg.name}: {cfg.description}", "slots_per_step": per_step,
                       "T": cfg.link.T, "F": cfg.link.F, "N": cfg.link.N},
            "cpu_baseline": {"value": v, "unit": "slots/s", "cores": threads, "kind": kind,
                             "sample": f"{per_step} slots per step (bounded sample of the {cfg.batch}-slot batch)"},
            "e2e": {"value": v, "unit": "slots/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--precision", default="")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-latency", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer leg (profiling runs only)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    from paper_2510_12739_b200 import graph as G
    cfg = G.CONFIGS[args.config]
    g = cfg.graph(seed=1)
    if args.impl == "reference":
        run_reference(args, cfg, g)
        return

    import torch
    import torch.distributed as dist
    from paper_2510_12739_b200 import plan as P, slots

    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    B = args.batch or cfg.batch
    prec = args.precision or cfg.precision
    link = cfg.link
    batch = slots.generate(link, B, seed=1000 + rank)
    plan = P.Plan(g, prec, device=local)
    plan.set_pilots(batch.pilots, batch.pilot_mask)
    nb = g.output_channels()
    stream = torch.cuda.Stream()
    st = stream.cuda_stream
    y_dev = torch.from_numpy(batch.y).cuda()
    out = torch.empty((B, link.T, link.F, nb), dtype=torch.float32, device="cuda")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    # ---------------- value leg: inputs resident in HBM ----------------
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            plan.receive_device(y_dev, out, st)
    torch.cuda.synchronize()

    def timed_steps(profile: bool):
        # K steps, the L2 flushed (untimed) before each; per-launch events only when profiling (an event
        # between two launches cancels their programmatic dependent launch, so `value` is timed without)
        plan.set_profiling(profile)
        plan.read_profile()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            with torch.cuda.stream(stream):
                for i in range(args.steps):
                    flush.fill_(i & 0xFF)
                    evs[i][0].record(stream)
                    plan.receive_device(y_dev, out, st)
                    evs[i][1].record(stream)
            torch.cuda.synchronize()
            barrier()
        plan.set_profiling(False)
        return sum(a.elapsed_time(b) for a, b in evs), plan.read_profile(), clk

    dev_ms, _, clk = timed_steps(False)
    # the same K steps again with per-launch events, for the dominant kernel's roofline
    prof_ms, prof, _ = timed_steps(True)
    dev_ms = max_over_ranks(dev_ms)
    value = world * B * args.steps / (dev_ms / 1e3)
    launches_per_step = len(plan.launch_names())

    # dominant kernel roofline (per-launch events in the timed region)
    info = plan.info()
    agg = {}
    for name, ms, cnt in prof:
        a = agg.setdefault(name, [0.0, 0])
        a[0] += ms
        a[1] += cnt
    top = max(agg.items(), key=lambda kv: kv[1][0])
    top_name, (top_ms, top_cnt) = top[0], top[1]
    flops_per_re = plan.launch_flops_per_re()
    top_flops = [f for (n, f) in zip(plan.launch_names(), flops_per_re) if n == top_name]
    res_per_step = B * link.T * link.F
    avg_launch_ms = top_ms / top_cnt
    achieved_tflops = (np.mean(top_flops) * res_per_step) / (avg_launch_ms * 1e-3) / 1e12 if top_flops else None
    peak_tf, peak_hbm, peak_src = peaks()
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get(top_name)
    share = top_ms / sum(v[0] for v in agg.values())

    # ---------------- e2e leg: C-ABI host call, pinned host buffers ----------------
    y_host = torch.from_numpy(batch.y).pin_memory()
    out_host = torch.empty((B, link.T, link.F, nb), dtype=torch.float32).pin_memory()
    for _ in range(0 if args.no_e2e else max(2, args.warmup // 2)):
        plan.receive_host_ptr(y_host.data_ptr(), batch.y.shape, out_host.data_ptr())
    e2e_steps = 0 if args.no_e2e else max(5, args.steps // 4)
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        plan.receive_host_ptr(y_host.data_ptr(), batch.y.shape, out_host.data_ptr())
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    barrier()
    e2e_value = world * B * e2e_steps / e2e_s if e2e_steps else None
    h2d = batch.y.nbytes
    d2h = out_host.numel() * 4

    # ---------------- B=1 latency (CUDA graph replay) ----------------
    lat = None
    if not args.no_latency:
        p1 = P.Plan(g, prec, device=local)
        p1.set_pilots(batch.pilots, batch.pilot_mask)
        p1.set_graph_capture(True)
        y1 = y_dev[:1].contiguous()
        o1 = torch.empty((1, link.T, link.F, nb), dtype=torch.float32, device="cuda")
        with torch.cuda.stream(stream):
            for _ in range(5):
                p1.receive_device(y1, o1, st)
        torch.cuda.synchronize()
        dev_lat = []
        for _ in range(200):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            p1.receive_device(y1, o1, st)
            b.record(stream)
            b.synchronize()
            dev_lat.append(a.elapsed_time(b))
        p1.set_graph_capture(False)
        yh1 = torch.from_numpy(batch.y[:1].copy()).pin_memory()
        oh1 = torch.empty((1, link.T, link.F, nb), dtype=torch.float32).pin_memory()
        for _ in range(5):
            p1.receive_host_ptr(yh1.data_ptr(), (1, link.T, link.F, link.N), oh1.data_ptr())
        e2e_lat = []
        for _ in range(200):
            t = time.perf_counter()
            p1.receive_host_ptr(yh1.data_ptr(), (1, link.T, link.F, link.N), oh1.data_ptr())
            e2e_lat.append((time.perf_counter() - t) * 1e3)
        lat = {"device_ms": {"p50": float(np.percentile(dev_lat, 50)), "p99": float(np.percentile(dev_lat, 99))},
               "e2e_ms": {"p50": float(np.percentile(e2e_lat, 50)), "p99": float(np.percentile(e2e_lat, 99))}}
        p1.close()

    # ---------------- CPU baseline (rank 0, N=1 only) ----------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(cfg, g, batch)
        except Exception as e:  # reported, never fatal for the GPU number
            cpu = {"value": None, "unit": "slots/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "slots/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": prec, "data": "synthetic",
            "res_per_s": value * link.T * link.F,
            "config": {"workload": f"{cfg.name}: {cfg.description}", "global_batch": B * world, "slots_per_gpu": B,
                       "T": link.T, "F": link.F, "N": link.N, "mod_order": link.mod_order,
                       "parallelism": f"slot-sharded x{world} (no data-path collective)",
                       "l2": "flushed between timed steps (256 MiB write, untimed)",
                       "flop_per_slot": 2.0 * g.macs_per_re() * link.T * link.F},
            "roofline": {"bound": "tensor", "kernel": top_name, "achieved": achieved_tflops, "peak": peak_tf,
                         "unit": "TFLOP/s", "frac": (achieved_tflops / peak_tf) if achieved_tflops else None,
                         "peak_source": peak_src + ", sustained bf16", "traffic": traffic,
                         "avg_launch_ms": avg_launch_ms, "launches_per_step": top_cnt // args.steps,
                         "share_of_step": share,
                         "timing": "per-launch CUDA events over a second pass of the K timed steps "
                                   f"({prof_ms / args.steps:.3f} ms/step with the events)",
                         "whole_step_tflops": 2.0 * g.macs_per_re() * res_per_step * args.steps / (dev_ms * 1e-3) / 1e12},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "slots/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "api": "cnrx_receive (C ABI, pinned host buffers)"},
            "latency_b1": lat,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
