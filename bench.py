"""CoNet-Rx batched inference benchmark (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg2]
                    [--strong [--total-batch 8192]] [--no-extra]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (BASELINE.json metric "CoNet-Rx inference slots/s and REs/s ... p50 per-slot latency",
quoted on configs[1] = cfg2): one step = featurize -> 3 ResNet subnetworks -> mul+BN fusion -> 1x1
LLR head over B=256 seeded synthetic slots per GPU (612 subcarriers x 14 symbols, 2 RX antennas,
16-QAM, TDL 12 taps / 300 ns / Jakes <= 200 Hz, SNR U[0,25] dB), bf16 plan (BASELINE's precision).
Slots are sharded across ranks with no data-path collective (weak scaling: B per GPU fixed; --strong:
cfg5's total batch split across the ranks).

  value   slots/s, inputs resident in HBM, device time (CUDA events on the launching stream), L2
          flushed (256 MiB write, untimed) before every timed step, max over ranks
  e2e     slots/s through the C-ABI host call cnrx_receive (pinned host y in, host LLRs out; H2D +
          D2H inside the timed region); at N > 1 the final LLR gather is inside it too: every rank
          receives its slot range on its GPU, the LLRs are gathered to rank 0's GPU over NCCL and rank
          0 copies the whole batch to its pinned host buffer
  roofline  dominant kernel: algorithmic FLOPs per launch (2 x MACs over all taps) /
          its average launch time from per-launch CUDA events over a second pass of the K timed
          steps (events between launches cancel programmatic dependent launch, so `value` is timed
          without them); peak = MEASURED_PEAKS.json burst bf16 when the SM clock sampled during the
          timed region stays within 5 % of max, the sustained figure otherwise (`peak_kind`)
  clocks  NVML SM clock + clock-event reasons sampled every 5 ms inside the timed region
  precision_variants  the same step on the FP16 plan (the option that meets the hard-decision bar) and on
          the BF16X3 split-precision plan (fp32-grade LLRs on the tensor cores)
  extra_configs (N = 1)  cfg1 (fp32 and bf16x3), cfg3 (bf16 / fp16 / bf16x3), cfg4 / cfg4m at their BASELINE
          batch, the cfg5 batch sweep (bf16 / fp16 / bf16x3 / fp32) with p50 latency at B = 1, each with its
          roofline and a CPU baseline
  cpu_baseline  the reference's own Network<float>::forward and forward_concurrent (oracle/_ref,
          compiled in place from /root/reference) + the restated featurizer, all host threads,
          median of 5 reps of a bounded sample
"""
from __future__ import annotations

import argparse
import json
import math
import os
import platform
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CoNet-Rx inference slots/s and REs/s at 1/2/4/8 B200; p50 per-slot latency"
SM_COUNT = 148


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return {"burst": d.get("bf16_tflops", 1639.2), "sustained": d.get("bf16_tflops_sustained", 1396.9),
                "hbm": d.get("hbm_gbs", 6547.2), "sm_max_mhz": d.get("sm_max_mhz", 1965.0),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"burst": 1590.0, "sustained": 1400.0, "hbm": 6650.0, "sm_max_mhz": 1965.0,
            "source": "fallback (B200_PROFILING.md)"}


def pick_peak(pk: dict, clocks: dict):
    """Burst bf16 peak when the timed region ran at (within 5 % of) max SM clock, else sustained."""
    med, mx = clocks.get("sm_mhz"), clocks.get("sm_max_mhz") or pk["sm_max_mhz"]
    if med is not None and med >= 0.95 * mx:
        return pk["burst"], "burst"
    return pk["sustained"], "sustained"


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


class ClockSampler:
    """NVML SM clock / clock-event reasons / power every `period` s on a thread while the timed region
    runs (nvidia-smi's 100 ms loop gave one sample over a 90 ms region)."""

    NAMES = {"nvmlClocksEventReasonSwPowerCap": "sw_power_cap", "nvmlClocksEventReasonHwSlowdown": "hw_slowdown",
             "nvmlClocksEventReasonHwThermalSlowdown": "hw_thermal_slowdown",
             "nvmlClocksEventReasonSwThermalSlowdown": "sw_thermal_slowdown",
             "nvmlClocksEventReasonHwPowerBrakeSlowdown": "hw_power_brake_slowdown",
             "nvmlClocksEventReasonSyncBoost": "sync_boost",
             "nvmlClocksEventReasonApplicationsClocksSetting": "applications_clocks_setting",
             "nvmlClocksEventReasonDisplayClockSetting": "display_clock_setting"}

    def __init__(self, cuda_index: int, period: float = 0.005):
        self.period = period
        self.samples = []
        self.h = None
        try:
            import pynvml as N
            import torch
            N.nvmlInit()
            self.N = N
            try:
                uuid = "GPU-" + str(torch.cuda.get_device_properties(cuda_index).uuid)
                self.h = N.nvmlDeviceGetHandleByUUID(uuid)
            except Exception:
                vis = os.environ.get("CUDA_VISIBLE_DEVICES")
                idx = int(vis.split(",")[cuda_index]) if vis and vis.split(",")[0].isdigit() else cuda_index
                self.h = N.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM))
        except Exception:
            self.h = None

    def __enter__(self):
        self.stop = threading.Event()
        if self.h is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def _run(self):
        N = self.N
        while not self.stop.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)
                rs = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                pw = N.nvmlDeviceGetPowerUsage(self.h) / 1000.0
                self.samples.append((float(sm), int(rs), pw))
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self.stop.set()
        if self.h is not None:
            self.t.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "source": "nvml unavailable"}
        sm = [s[0] for s in self.samples]
        reasons = set()
        for _, bits, _ in self.samples:
            for attr, name in self.NAMES.items():
                v = getattr(self.N, attr, None)
                if v is not None and bits & v:
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)), "sm_min_mhz": float(min(sm)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(sm), "power_w": float(np.median([s[2] for s in self.samples])),
                "source": f"NVML every {self.period * 1e3:.0f} ms inside the timed region"}


# ------------------------------------------------------------------------------------------------
# CPU baseline: the reference's own forward on this host
# ------------------------------------------------------------------------------------------------
def ref_forward_fn(g):
    import oracle
    os.environ.setdefault("CONETRX_THREADS", str(os.cpu_count() or 1))
    os.environ.pop("CONETRX_DETERMINISTIC", None)
    if oracle.ref_available():
        net = oracle.RefNet.from_graph(g)
        return "reference", int(oracle.ref().ref_threads()), (lambda x, conc=False: net.forward(x, concurrent=conc))
    return "port", 1, (lambda x, conc=False: oracle.forward(g, x))


def cpu_baseline(cfg, g, batch, n_slots, reps=5, f_sample=None):
    """Median of `reps` reps over `n_slots` slots (featurize + Network<float>::forward, and
    forward_concurrent): slots/s.  f_sample: time a sub-grid of that many subcarriers and scale per RE
    (for cfg3, where one full slot takes seconds per core)."""
    import copy
    import oracle
    note = ""
    if any(n.dilation_f != 1 for n in g.nodes):
        # the reference conv2d has no dilation (kernels.hpp:70-75): time the same graph at dilation 1,
        # which does the same work per RE (every tap computed, out-of-grid taps skipped either way)
        g = copy.deepcopy(g)
        for n in g.nodes:
            n.dilation_f = 1
        note = "; graph timed at dilation 1 (the reference conv has none; same work per RE)"
    kind, threads, fwd = ref_forward_fn(g)
    y = batch.y[:n_slots]
    pil, pm = batch.pilots, batch.pilot_mask
    scale = 1.0
    if f_sample and f_sample < y.shape[2]:
        y, pil, pm = y[:, :, :f_sample], pil[:, :f_sample], pm[:, :f_sample]
        scale = f_sample / batch.y.shape[2]
    res = {}
    for conc in (False, True):
        if kind == "port" and conc:
            continue
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fwd(oracle.featurize(y, pil, pm), conc)
            ts.append(time.perf_counter() - t0)
        res["forward_concurrent" if conc else "forward"] = n_slots * scale / float(np.median(ts))
    best = max(res, key=res.get)
    samp = f"{n_slots} {cfg.name} slots" + (f" (sub-grid F={f_sample} of {batch.y.shape[2]}, scaled per RE)" if scale < 1 else "")
    return {"value": res[best], "unit": "slots/s", "cores": threads, "kind": kind,
            "cpu": f"{cpu_model()}, {os.cpu_count()} logical CPUs",
            "per_call": {k: round(v, 4) for k, v in res.items()}, "best_call": best,
            "sample": f"median of {reps} reps of {samp}: restated featurize + reference Network<float>::"
                      f"forward / forward_concurrent (eval), CONETRX_THREADS={os.environ.get('CONETRX_THREADS')}{note}"}


def run_reference(args, cfg, g):
    rank, local, world = dist_env()
    if rank != 0:
        return
    from paper_2510_12739_b200 import slots
    import oracle
    cores = os.cpu_count() or 1
    per_step = max(1, min(cfg.batch, cores))
    batch = slots.generate(cfg.link, per_step, seed=1000)
    kind, threads, fwd = ref_forward_fn(g)

    def step():
        fwd(oracle.featurize(batch.y, batch.pilots, batch.pilot_mask), False)

    for _ in range(args.warmup):
        step()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        ts.append(time.perf_counter() - t0)
    dt = sum(ts)
    v = per_step * args.steps / dt
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "slots/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "res_per_s": v * cfg.link.T * cfg.link.F,
            "config": {"workload": f"{cfg.name}: {cfg.description}", "slots_per_step": per_step,
                       "T": cfg.link.T, "F": cfg.link.F, "N": cfg.link.N},
            "cpu_baseline": {"value": v, "unit": "slots/s", "cores": threads, "kind": kind,
                             "cpu": f"{cpu_model()}, {cores} logical CPUs",
                             "sample": f"{per_step} slots per step (bounded sample of the {cfg.batch}-slot batch), "
                                       f"median step {np.median(ts) * 1e3:.0f} ms"},
            "e2e": {"value": v, "unit": "slots/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------
# device timing helpers
# ------------------------------------------------------------------------------------------------
class Leg:
    """One plan + resident inputs; timed steps with the L2 flushed before each."""

    def __init__(self, torch, P, g, prec, batch, link, device, options=None):
        self.torch = torch
        self.prec = prec
        self.plan = P.Plan(g, prec, device=device, options=options)
        self.plan.set_pilots(batch.pilots, batch.pilot_mask)
        self.B = batch.y.shape[0]
        self.link = link
        self.nb = g.output_channels()
        self.stream = torch.cuda.Stream()
        self.y = torch.from_numpy(batch.y).cuda()
        self.out = torch.empty((self.B, link.T, link.F, self.nb), dtype=torch.float32, device="cuda")
        self.flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    def run(self):
        self.plan.receive_device(self.y, self.out, self.stream.cuda_stream)

    def warm(self, n):
        with self.torch.cuda.stream(self.stream):
            for _ in range(n):
                self.run()
        self.torch.cuda.synchronize()

    def timed(self, steps, profile=False, clock_index=None, barrier=lambda: None):
        torch = self.torch
        self.plan.set_profiling(profile)
        self.plan.read_profile()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        barrier()
        torch.cuda.synchronize()
        clk = ClockSampler(clock_index) if clock_index is not None else None
        if clk:
            clk.__enter__()
        try:
            with torch.cuda.stream(self.stream):
                for i in range(steps):
                    self.flush.fill_(i & 0xFF)
                    evs[i][0].record(self.stream)
                    self.run()
                    evs[i][1].record(self.stream)
            torch.cuda.synchronize()
        finally:
            if clk:
                clk.__exit__()
        barrier()
        self.plan.set_profiling(False)
        ms = [a.elapsed_time(b) for a, b in evs]
        return ms, (self.plan.read_profile() if profile else None), (clk.summary() if clk else None)

    def roofline(self, prof, steps, pk, clocks, bound="tensor"):
        """Dominant kernel by summed per-launch time: algorithmic FLOPs per launch / mean launch time."""
        agg = {}
        for name, ms, cnt in prof:
            a = agg.setdefault(name, [0.0, 0])
            a[0] += ms
            a[1] += cnt
        top_name, (top_ms, top_cnt) = max(agg.items(), key=lambda kv: kv[1][0])
        names, fl = self.plan.launch_names(), self.plan.launch_flops_per_re()
        top_flops = [f for n, f in zip(names, fl) if n == top_name]
        res = self.B * self.link.T * self.link.F
        avg_ms = top_ms / top_cnt
        # algorithmic work of the kernel per step / its device time per step.  `top_flops` lists the
        # kernel's launches in one pass of the program; batches beyond the plan's memory budget run the
        # program once per slot chunk (launches_per_step > len(top_flops)) over the same REs in total.
        work = float(np.sum(top_flops)) * res if top_flops else 0.0
        achieved = work / (top_ms / steps * 1e-3) / 1e12 if work > 0 else None
        out = {"kernel": top_name, "avg_launch_ms": avg_ms, "launches_per_step": top_cnt // steps,
               "share_of_step": top_ms / sum(v[0] for v in agg.values()),
               "algorithmic_tflop_per_launch": work / (top_cnt // steps) / 1e12 if top_flops else None,
               "slot_chunks": max(1, (top_cnt // steps) // max(1, len(top_flops)))}
        if bound == "ffma":  # fp32 CUDA-core plans: nominal FP32 FMA peak at the sampled SM clock
            mhz = (clocks or {}).get("sm_mhz") or pk["sm_max_mhz"]
            peak = SM_COUNT * 128 * 2 * mhz * 1e6 / 1e12
            out.update({"bound": "ffma", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                        "frac": achieved / peak if achieved else None,
                        "peak_kind": f"nominal FP32 (148 SMs x 128 FMA/clk) at the sampled {mhz:.0f} MHz",
                        # the reference's arithmetic is a separately rounded multiply then add (no FMA):
                        # two FP32 lane-ops per MAC, measured 62 MAC/clk/SM (tools/probes/ffma2_probe.cu)
                        "bit_exact_peak": peak / 2,
                        "frac_of_bit_exact_peak": 2 * achieved / peak if achieved else None})
        else:
            peak, kind = pick_peak(pk, clocks or {})
            out.update({"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                        "frac": achieved / peak if achieved else None,
                        "peak_kind": f"{kind} bf16 ({pk['source']}); the fp16 kind::f16 rate is the same"})
            if self.prec.endswith("x3"):
                # split-precision plans: every MAC is three 16-bit tensor-core products (hi*Whi + lo*Whi +
                # hi*Wlo); `achieved` counts the algorithmic (fp32) FLOPs, `issued_frac` the tensor pipe's
                out.update({"tensor_products_per_mac": 3, "issued_frac": 3 * achieved / peak if achieved else None})
        return out

    def close(self):
        self.plan.close()
        del self.y, self.out, self.flush


def measure_config(torch, P, G, slots, name, prec, B, steps, warmup, local, pk, seed=77, want_cpu=True,
                   cpu_slots=8, f_sample=None):
    """One BASELINE config at batch B on this GPU: device ms/step (median of `steps`), slots/s, roofline
    of its dominant kernel, clocks, and (optionally) the reference CPU forward on a bounded sample."""
    cfg = G.CONFIGS[name]
    g = cfg.graph(seed=1)
    batch = slots.generate(cfg.link, B, seed=seed)
    leg = Leg(torch, P, g, prec, batch, cfg.link, local, options={})
    leg.warm(warmup)
    ms, _, clk = leg.timed(steps, clock_index=local)
    _, prof, _ = leg.timed(max(2, steps // 2), profile=True)
    med = float(np.median(ms))
    r = {"config": name, "precision": prec, "batch": B, "ms_per_step_median": med,
         "ms_per_step_min": float(min(ms)), "steps": steps,
         "slots_per_s": B / (med * 1e-3), "res_per_s": B * cfg.link.T * cfg.link.F / (med * 1e-3),
         "whole_step_tflops": 2.0 * g.macs_per_re() * B * cfg.link.T * cfg.link.F / (med * 1e-3) / 1e12,
         "roofline": leg.roofline(prof, max(2, steps // 2), pk, clk, bound="ffma" if prec == "fp32" else "tensor"),
         "clocks": clk, "launches_per_step": len(leg.plan.launch_names())}
    leg.close()
    torch.cuda.empty_cache()
    if want_cpu:
        try:
            r["cpu_baseline"] = cpu_baseline(cfg, g, batch, min(cpu_slots, B), reps=5, f_sample=f_sample)
        except Exception as e:
            r["cpu_baseline"] = {"value": None, "sample": f"unavailable: {e}"}
    return r


def latency_b1(torch, P, g, prec, batch, link, local):
    p1 = P.Plan(g, prec, device=local, options={})
    p1.set_pilots(batch.pilots, batch.pilot_mask)
    p1.set_graph_capture(True)
    nb = g.output_channels()
    stream = torch.cuda.Stream()
    st = stream.cuda_stream
    y1 = torch.from_numpy(batch.y[:1].copy()).cuda()
    o1 = torch.empty((1, link.T, link.F, nb), dtype=torch.float32, device="cuda")
    with torch.cuda.stream(stream):
        for _ in range(5):
            p1.receive_device(y1, o1, st)
    torch.cuda.synchronize()
    dev_lat = []
    # one synchronous replay at a time leaves the GPU mostly idle: the SM clock during these runs is what the
    # driver's idle governor gives (it scales the latency ~1/clock), so it is sampled and reported with them
    with ClockSampler(local) as cs:
        for _ in range(200):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            p1.receive_device(y1, o1, st)
            b.record(stream)
            b.synchronize()
            dev_lat.append(a.elapsed_time(b))
    lat_clocks = cs.summary()
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
    p1.close()
    return {"device_ms": {"p50": float(np.percentile(dev_lat, 50)), "p99": float(np.percentile(dev_lat, 99))},
            "e2e_ms": {"p50": float(np.percentile(e2e_lat, 50)), "p99": float(np.percentile(e2e_lat, 99))},
            "device_clocks": {k: lat_clocks.get(k) for k in ("sm_mhz", "sm_min_mhz", "sm_max_mhz", "samples")},
            "how": "B=1, 200 runs; device: CUDA-graph replay between CUDA events; e2e: cnrx_receive from pinned host"}


def extra_configs(torch, P, G, slots, local, pk, steps):
    """Driver-visible numbers for the other BASELINE configs, N = 1."""
    out = {}
    k = max(3, min(steps, 10))
    def one(key, *a, **kw):  # a failing config is recorded, the others still run
        try:
            out[key] = measure_config(torch, P, G, slots, *a, **kw)
        except Exception as e:
            out[key] = {"error": repr(e)}
            torch.cuda.empty_cache()

    one("cfg1_fp32_b64", "cfg1", "fp32", 64, k, 3, local, pk, cpu_slots=64)
    # the fp32-grade tensor-core plan (LLRs within 1e-4 of the reference) on the fp32 config
    one("cfg1_bf16x3_b64", "cfg1", "bf16x3", 64, k, 3, local, pk, want_cpu=False)
    one("cfg3_bf16x3_b64", "cfg3", "bf16x3", 64, 3, 2, local, pk, want_cpu=False)
    for prec in ("bf16", "fp16"):
        one(f"cfg3_{prec}_b64", "cfg3", prec, 64, k, 3, local, pk, want_cpu=prec == "bf16", cpu_slots=16, f_sample=137)
    one("cfg4_bf16_b256", "cfg4", "bf16", 256, k, 3, local, pk, cpu_slots=8)
    one("cfg4m_bf16_b256", "cfg4m", "bf16", 256, k, 3, local, pk, cpu_slots=8)
    # cfg5: the cfg2 batch sweep, bf16 / fp16 tensor-core plans, the fp32-grade split-precision tensor-core
    # plan (bf16x3) and the bit-exact fp32 CUDA-core plan
    sweep = []
    cfg = G.CONFIGS["cfg2"]
    g = cfg.graph(seed=1)
    for prec, Bs in (("bf16", (1, 4, 16, 64, 256, 1024, 4096, 8192)), ("fp16", (1, 64, 256, 1024, 8192)),
                     ("bf16x3", (1, 16, 256, 1024, 8192)), ("fp32", (1, 16, 256, 1024))):
        for B in Bs:
            kk = 3 if (prec in ("fp32", "bf16x3") and B >= 256) or B >= 4096 else k
            try:
                r = measure_config(torch, P, G, slots, "cfg2", prec, B, kk, 2, local, pk, want_cpu=False)
            except Exception as e:  # recorded per point, never fatal for the rest of the sweep
                sweep.append({"precision": prec, "batch": B, "error": repr(e)})
                torch.cuda.empty_cache()
                continue
            sweep.append({kk2: r[kk2] for kk2 in ("precision", "batch", "ms_per_step_median", "slots_per_s",
                                                   "res_per_s", "whole_step_tflops")} |
                         {"roofline_frac": r["roofline"]["frac"], "roofline_kernel": r["roofline"]["kernel"],
                          "sm_mhz": (r["clocks"] or {}).get("sm_mhz")})
        batch = slots.generate(cfg.link, 1, seed=5)
        sweep.append({"precision": prec, "batch": 1, "latency_b1": latency_b1(torch, P, g, prec, batch, cfg.link, local)})
    out["cfg5_sweep"] = sweep
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--batch", type=int, default=0, help="slots per GPU (weak scaling)")
    ap.add_argument("--strong", action="store_true", help="cfg5 strong scaling: --total-batch split across ranks")
    ap.add_argument("--total-batch", type=int, default=8192)
    ap.add_argument("--precision", default="")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-latency", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer leg (profiling runs only)")
    ap.add_argument("--no-extra", action="store_true", help="skip extra_configs / precision variants")
    ap.add_argument("--gather", default="peer", choices=["peer", "nccl"],
                    help="N > 1 e2e: LLRs stored into rank 0's buffer by each rank's head kernel over NVLink "
                         "(peer, default) or an NCCL gather after the forward")
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
    # flow test of the multi-rank path on a one-GPU box only (never a measurement): every rank on cuda:0,
    # gloo plumbing (NCCL refuses two ranks on one GPU)
    share = os.environ.get("CNRX_BENCH_SHARE_GPU") == "1"
    backend = "gloo" if share else "nccl"
    if share:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    if args.strong:
        B = math.ceil(args.total_batch / world)
        global_batch = B * world
    else:
        B = args.batch or cfg.batch
        global_batch = B * world
    prec = args.precision or cfg.precision
    link = cfg.link
    pk = peaks()
    batch = slots.generate(link, B, seed=1000 + rank)
    nb = g.output_channels()

    # ---------------- value leg: inputs resident in HBM ----------------
    leg = Leg(torch, P, g, prec, batch, link, local, options={})
    leg.warm(args.warmup)
    ms, _, clk = leg.timed(args.steps, clock_index=local, barrier=barrier)
    dev_ms = max_over_ranks(sum(ms))
    value = global_batch * args.steps / (dev_ms / 1e3)
    launches_per_step = len(leg.plan.launch_names())
    # the same K steps again with per-launch events, for the dominant kernel's roofline
    pms, prof, _ = leg.timed(args.steps, profile=True, barrier=barrier)
    roof = leg.roofline(prof, args.steps, pk, clk)
    roof["timing"] = (f"per-launch CUDA events over a second pass of the K timed steps "
                      f"({sum(pms) / args.steps:.3f} ms/step with the events vs {sum(ms) / args.steps:.3f} without)")
    roof["whole_step_tflops"] = 2.0 * g.macs_per_re() * B * link.T * link.F * args.steps / (sum(ms) * 1e-3) / 1e12
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    roof["traffic"] = None
    if os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
        roof["traffic"] = tj.get(roof["kernel"].split("<")[0]) or tj.get(roof["kernel"])
        roof["traffic_source"] = tj.get("_source", "profiles/ncu_traffic.json") + " (carried over: ncu cannot run inside the timed bench)"
    # sustained: a longer run of the same step (the driver's K is a short burst at boost clock)
    sus = None
    if rank == 0 and world == 1 and not args.no_extra:
        sms, _, sclk = leg.timed(max(200, args.steps), clock_index=local)
        sus = {"value": B * len(sms) / (sum(sms) * 1e-3), "steps": len(sms), "clocks": sclk,
               "ms_per_step": float(np.mean(sms))}
    leg.close()
    torch.cuda.empty_cache()

    # ---------------- e2e leg: C-ABI host call, pinned host buffers (+ LLR gather at N > 1) ----------------
    e2e = None
    if not args.no_e2e:
        plan = P.Plan(g, prec, device=local, options={})
        plan.set_pilots(batch.pilots, batch.pilot_mask)
        y_host = torch.from_numpy(batch.y).pin_memory()
        if world == 1:
            out_host = torch.empty((B, link.T, link.F, nb), dtype=torch.float32).pin_memory()

            def e2e_step():
                plan.receive_host_ptr(y_host.data_ptr(), batch.y.shape, out_host.data_ptr())
            h2d, d2h = batch.y.nbytes, out_host.numel() * 4
            how = "cnrx_receive (C ABI, pinned host buffers, batch pipelined in chunks over two copy streams)"
        gather = args.gather
        if world > 1 and gather == "peer":
            try:  # collective: every rank agrees on the outcome
                from paper_2510_12739_b200 import shard as _shp
                # two buffers, alternating by step: rank 0 reads step k's batch while the other ranks' step
                # k + 1 stores go to the other buffer; the barrier of step k + 1 orders rank 0's read of
                # buffer k % 2 before anybody's step k + 2 stores into it
                peers = [_shp.PeerLLR(world * B, (link.T, link.F, nb), rank, local) for _ in range(2)]
            except RuntimeError as e:
                gather, peer_err = "nccl", repr(e)  # no peer access: the NCCL gather instead
        if world == 1:
            pass
        elif gather == "peer":
            # the final gather fused into the LLR head: rank 0's batch buffer is mapped into every rank (CUDA
            # IPC) and each rank's head kernel stores its slots straight into it over NVLink; completion =
            # stream sync + host barrier; rank 0 then reads the whole batch (one D2H)
            from paper_2510_12739_b200 import shard
            y_dev = torch.empty((B, link.T, link.F, link.N), dtype=torch.complex64, device="cuda")
            out_hosts = ([torch.empty((world * B, link.T, link.F, nb), dtype=torch.float32).pin_memory()
                          for _ in range(2)] if rank == 0 else None)
            out_host = out_hosts[0] if rank == 0 else None
            rd_stream = torch.cuda.Stream() if rank == 0 else None  # rank 0's D2H of step k overlaps step k + 1
            rd_done = [None, None]
            peer_step = [0]

            def e2e_step():
                k = peer_step[0] & 1
                peer = peers[k]
                peer_step[0] += 1
                y_dev.copy_(y_host, non_blocking=True)
                plan.receive_device_ptr(y_dev, peer.dst(rank * B), torch.cuda.current_stream().cuda_stream)
                torch.cuda.current_stream().synchronize()
                if rank == 0 and rd_done[k ^ 1] is not None:
                    # the previous step's read (of the other peer buffer) is complete before this barrier releases
                    # the ranks into the step that stores into that buffer again
                    rd_done[k ^ 1].synchronize()
                barrier()
                if rank == 0:
                    peer.to_host_async(out_hosts[k], rd_stream.cuda_stream)
                    rd_done[k] = torch.cuda.Event()
                    rd_done[k].record(rd_stream)

            def e2e_finish():  # inside the timed region: the last steps' reads have landed
                if rank == 0:
                    rd_stream.synchronize()
            h2d, d2h = batch.y.nbytes * world, world * B * link.T * link.F * nb * 4
            how = ("per rank: H2D + cnrx_receive_device whose LLR head stores its slots into rank 0's buffer over "
                   "NVLink (CUDA IPC peer memory: the gather fused into the last kernel, no collective); stream "
                   "sync + barrier; rank 0 D2H of the whole batch on a side stream (two peer buffers alternate by "
                   "step, so rank 0's read of step k overlaps step k + 1 without its stores landing in the buffer "
                   "being read; the last reads complete inside the timed region)")
        else:
            # every rank: H2D of its slots, receive on its GPU; NCCL gather of the LLRs to rank 0's GPU
            # (shard.gather_llr_tensor, covered by the 2-rank gloo test); rank 0: one D2H of the whole
            # batch into its pinned host buffer
            from paper_2510_12739_b200 import shard
            y_dev = torch.empty((B, link.T, link.F, link.N), dtype=torch.complex64, device="cuda")
            out_dev = torch.empty((B, link.T, link.F, nb), dtype=torch.float32, device="cuda")
            out_host = torch.empty((world * B, link.T, link.F, nb), dtype=torch.float32).pin_memory() if rank == 0 else None

            def e2e_step():
                y_dev.copy_(y_host, non_blocking=True)
                plan.receive_device(y_dev, out_dev, torch.cuda.current_stream().cuda_stream)
                if backend == "nccl":
                    full = shard.gather_llr_tensor(out_dev, world * B, world, rank)
                else:  # flow test (CNRX_BENCH_SHARE_GPU): gloo gathers host tensors
                    full = shard.gather_llr_tensor(out_dev.cpu(), world * B, world, rank)
                if rank == 0:
                    out_host.copy_(full, non_blocking=True)
                torch.cuda.synchronize()
            h2d, d2h = batch.y.nbytes * world, world * B * link.T * link.F * nb * 4
            how = "per rank: H2D + cnrx_receive_device; NCCL gather of the LLRs to rank 0; rank 0 D2H of the whole batch"
        if not (world > 1 and gather == "peer"):
            def e2e_finish():
                pass
        for _ in range(max(2, args.warmup // 2)):
            e2e_step()
        e2e_finish()
        e2e_steps = max(5, args.steps // 4)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        e2e_finish()
        e2e_s = max_over_ranks(time.perf_counter() - t0)
        barrier()
        e2e = {"value": global_batch * e2e_steps / e2e_s, "unit": "slots/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "api": how, "steps": e2e_steps}
        if world > 1:
            e2e["nccl_ranks" if backend == "nccl" else "gloo_ranks_flow_test"] = dist.get_world_size()
            e2e["gather"] = gather
            if gather != args.gather:
                e2e["gather_fallback"] = peer_err
            if gather == "peer":
                # the peer-written batch equals the ranks' own LLRs gathered by the process group
                mine = torch.empty((B, link.T, link.F, nb), dtype=torch.float32, device="cuda")
                plan.receive_device(y_dev, mine, torch.cuda.current_stream().cuda_stream)
                torch.cuda.synchronize()
                from paper_2510_12739_b200 import shard as _sh
                ref = _sh.gather_llr_tensor(mine if backend == "nccl" else mine.cpu(), world * B, world, rank)
                if rank == 0:
                    e2e["peer_gather_bit_exact"] = bool(torch.equal(ref.cpu(), out_hosts[0]) and
                                                        torch.equal(ref.cpu(), out_hosts[1]))
                barrier()
                for peer in peers:
                    peer.close()
        plan.close()

    lat = None
    if not args.no_latency and rank == 0:
        lat = latency_b1(torch, P, g, prec, batch, link, local)

    # ---------------- FP16 plan: same step, the option that meets the decision bar ----------------
    variants = None
    if not args.no_extra and world == 1 and prec == "bf16":
        v = Leg(torch, P, g, "fp16", batch, link, local, options={})
        v.warm(args.warmup)
        vms, _, vclk = v.timed(args.steps, clock_index=local)
        _, vprof, _ = v.timed(args.steps, profile=True)
        variants = {"fp16": {"value": B * args.steps / (sum(vms) * 1e-3), "ms_per_step": sum(vms) / args.steps,
                             "roofline": v.roofline(vprof, args.steps, pk, vclk), "clocks": vclk,
                             "decision_agreement": "tests/test_trained.py (>= 99.99 % of all data bits vs fp32)"}}
        v.close()
        torch.cuda.empty_cache()
        # the split-precision plan: fp32-grade LLRs (<= 1e-4 relative of the reference) on the tensor cores
        v = Leg(torch, P, g, "bf16x3", batch, link, local, options={})
        v.warm(args.warmup)
        vms, _, vclk = v.timed(args.steps, clock_index=local)
        _, vprof, _ = v.timed(args.steps, profile=True)
        variants["bf16x3"] = {"value": B * args.steps / (sum(vms) * 1e-3), "ms_per_step": sum(vms) / args.steps,
                              "roofline": v.roofline(vprof, args.steps, pk, vclk), "clocks": vclk,
                              "parity": "tests/test_gpu_x3.py (<= 1e-4 relative of the reference); decisions "
                                        ">= 99.99 % on trained cfg2 and cfg3 (tests/test_trained.py)"}
        v.close()
        torch.cuda.empty_cache()

    # ---------------- CPU baseline (rank 0, N=1 only) ----------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(cfg, g, batch, min(B, max(8, (os.cpu_count() or 8))), reps=5)
        except Exception as e:  # reported, never fatal for the GPU number
            cpu = {"value": None, "unit": "slots/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    extra = None
    if rank == 0 and world == 1 and not args.no_extra:
        try:
            extra = extra_configs(torch, P, G, slots, local, pk, args.steps)
        except Exception as e:
            extra = {"error": repr(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "slots/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": prec,
            "data": "synthetic", "res_per_s": value * link.T * link.F,
            "config": {"workload": f"{cfg.name}: {cfg.description}", "global_batch": global_batch, "slots_per_gpu": B,
                       "T": link.T, "F": link.F, "N": link.N, "mod_order": link.mod_order,
                       "parallelism": f"slot-sharded x{world} (no data-path collective; LLR gather in e2e)",
                       "l2": "flushed between timed steps (256 MiB write, untimed)",
                       "flop_per_slot": 2.0 * g.macs_per_re() * link.T * link.F},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "latency_b1": lat,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk,
            "sustained": sus,
            "precision_variants": variants,
            "extra_configs": extra,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
