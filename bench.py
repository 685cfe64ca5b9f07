#!/usr/bin/env python
"""bench.py — MoE-layer tokens/s + p99 layer latency, Mixtral-8x7B shape, on B200.

Workload (BASELINE.json configs[1], "cfg2"): one MoE layer, 8 experts, top-2,
d_model 4096, d_ff 14336, 16384 tokens per GPU, Zipf(1.2)-skewed routing,
straggler replicas from the MoEless planner (scale_experts + place_experts on
each iteration's actual loads, memory cap = 4 extra replicas).  A "step" is
one full layer forward: gate -> plan -> replica-aware dispatch -> SwiGLU
grouped GEMM (tcgen05) -> combine, every step re-routed (new iteration index:
new token batch from a pool of 4 and a new gate noise permutation).

  python bench.py [--gpus N --steps K --warmup W]          # our sm_100a path
  python bench.py --impl reference [...]                   # CPU reference arm
  torchrun --nproc-per-node N bench.py --gpus N ...        # N > 1: expert parallel,
                                                           # weak scaling (16384 tokens/GPU)

Timing: W untimed warm-up steps, then exactly K steps bracketed by a barrier
+ cuda synchronize on both sides, CUDA events on the stream the kernels run
on, max over ranks.  Inputs (2.8 GB of weights, 134 MB of tokens per step)
are far larger than the 126 MB L2.  `e2e` repeats the measurement through the
C-ABI's host-buffer entry point (moe_layer_forward_host: H2D of x from pinned
memory + forward + D2H of y inside the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = dict(E=8, k=2, d=4096, ff=14336, T=16384, s=1.2, extra_replicas=4, seed=1)
METRIC = "MoE-layer tokens/s + p99 layer latency, Mixtral-8x7B shape, 1/2/4/8 B200"
WORKLOAD = ("cfg2: Mixtral-8x7B MoE layer (E=8, top-2, d_model=4096, d_ff=14336), "
            "16384 tokens per GPU, Zipf s=1.2 routing, straggler replicas (MoEless planner, "
            "cap 4 extra replicas), expert parallel over the GPUs")
# --workload: the other BASELINE.json layer shapes through the same flow (the
# headline metric is cfg2's; these lines are labelled with their own shape)
OTHER_WORKLOADS = {
    "cfg1": (dict(E=8, k=2, d=1024, ff=3584, T=2048, s=1.2, extra_replicas=0, seed=1),
             "cfg1: E=8 top-2 d_model=1024 d_ff=3584, 2048 tokens per GPU, Zipf s=1.2"),
    "cfg3": (dict(E=16, k=2, d=4096, ff=6400, T=16384, s=1.2, extra_replicas=8, seed=1),
             "cfg3: Phi-3.5-MoE layer (E=16, top-2, d_model=4096, d_ff=6400), 16384 tokens per GPU, Zipf s=1.2, "
             "expert parallel with straggler replicas"),
    "cfg5": (dict(E=64, k=8, d=2048, ff=1408, T=256, s=2.0, extra_replicas=16, seed=1),
             "cfg5: fine-grained decode (E=64, top-8, d_model=2048, d_ff=1408), 256 tokens per GPU, heavy skew "
             "Zipf s=2.0"),
    "cfg5s12": (dict(E=64, k=8, d=2048, ff=1408, T=256, s=1.2, extra_replicas=16, seed=1),
                "cfg5 at the milder skew: fine-grained decode (E=64, top-8, d_model=2048, d_ff=1408), 256 tokens "
                "per GPU, Zipf s=1.2"),
}
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)   # p99 over >= 200 timed layers
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--pool", type=int, default=4, help="distinct token batches cycled per rank")
    ap.add_argument("--cpu-sample-tokens", type=int, default=4096,
                    help="tokens of the step's batch the reference arm runs per step (~2-4 s of host work)")
    ap.add_argument("--cpu-full-layer", type=int, default=1,
                    help="reference arm: also time one full-batch layer after the steps (0: skip)")
    ap.add_argument("--cpu-baseline-tokens", type=int, default=1024,
                    help="tokens per sample of our arm's cpu_baseline leg (two samples)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", choices=["p2p", "nccl"], default="p2p",
                    help="N>1 token exchange: peer memory over NVLink (dispatch/combine read and write the "
                         "owners' buffers) or NCCL grouped send/recv")
    ap.add_argument("--workload", choices=["cfg2", "cfg1", "cfg3", "cfg5", "cfg5s12"], default="cfg2",
                    help="layer shape (cfg2 = the headline Mixtral layer)")
    ap.add_argument("--plan", choices=["sync", "predicted"], default=None,
                    help="sync: scale/place on each step's actual loads (a host round trip per layer at N>1); "
                         "predicted: MoEless planning off the critical path (the layer's historical bootstrap "
                         "plans its next forward, which then runs device-planned).  Default: sync at N=1 (no "
                         "round trip there: the planner bookkeeping is deferred), predicted at N>1")
    ap.add_argument("--residency", choices=["all", "placed"], default="all",
                    help="N>1 expert weights: every expert resident on every GPU, or only home experts + "
                         "replica cache slots with cold replicas copied from their home GPU over NVLink")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d, "measured (MEASURED_PEAKS.json)"
    except Exception:
        return dict(FALLBACK_PEAKS), "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """dram bytes per GEMM launch from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "ncu_gemm_summary.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return None


class ClockSampler:
    """SM clocks and throttle reasons sampled with NVML every 20 ms in a
    background thread DURING the timed region (nvidia-smi's fields: clocks.sm,
    clocks.max.sm, power.draw, clocks_event_reasons.*)."""

    REASONS = (("nvmlClocksEventReasonHwSlowdown", "hw_slowdown"),
               ("nvmlClocksEventReasonHwThermalSlowdown", "hw_thermal_slowdown"),
               ("nvmlClocksEventReasonSwThermalSlowdown", "sw_thermal_slowdown"),
               ("nvmlClocksEventReasonSwPowerCap", "sw_power_cap"),
               ("nvmlClocksEventReasonHwPowerBrakeSlowdown", "hw_power_brake_slowdown"))

    def __init__(self, gpu_index, period_s=0.01):
        self.gpu, self.period = gpu_index, period_s
        self.rows, self.err = [], None
        self.e0 = self.energy_j = self.limit_w = None

    def _loop(self):
        import pynvml as N
        try:
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.gpu)
            smax = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            try:
                self.limit_w = N.nvmlDeviceGetEnforcedPowerLimit(h) / 1000.0
                self.e0 = N.nvmlDeviceGetTotalEnergyConsumption(h)  # mJ since driver load
            except Exception:  # noqa: BLE001 - energy counters are optional
                self.e0 = None
            while not self.stop.is_set():
                reasons = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append(dict(sm=N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM), smax=smax,
                                      power=N.nvmlDeviceGetPowerUsage(h) / 1000.0, reasons=reasons))
                self.ready.set()
                self.stop.wait(self.period)
            if self.e0 is not None:
                self.energy_j = (N.nvmlDeviceGetTotalEnergyConsumption(h) - self.e0) / 1000.0
        except Exception as e:  # no NVML: report unsampled
            self.err = repr(e)
        finally:
            self.ready.set()

    def __enter__(self):
        import threading
        self.stop = threading.Event()
        self.ready = threading.Event()
        self.th = threading.Thread(target=self._loop, daemon=True)
        self.th.start()
        self.ready.wait(timeout=10)  # NVML initialised and sampling before the timed region starts
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(timeout=5)

    def summary(self):
        import pynvml as N
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0, "error": self.err}
        # every sample lies inside the timed region (NVML power is a ~1 s
        # average, so it is not used to select "loaded" samples)
        loaded = self.rows
        reasons = set()
        for r in loaded:
            for attr, name in self.REASONS:
                if r["reasons"] & getattr(N, attr, 0):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(r["sm"] for r in loaded), "sm_max_mhz": max(r["smax"] for r in self.rows),
                "reasons": sorted(reasons), "samples": len(loaded),
                "power_w_median": statistics.median(r["power"] for r in loaded), "power_limit_w": self.limit_w,
                "energy_j": self.energy_j, "source": "NVML, 10 ms period; energy = total-energy counter delta"}


def nearest_rank(values, q):
    from paper_2603_06350_b200 import percentile
    return percentile(values, q)


def single_gpu_launches(T, k, E, d=4096):
    """Kernels of one G = 1 forward (capi.cpp enqueue_forward, default knobs)."""
    nblk = (T + 31) // 32
    swap = T * k / E <= 1024             # swap-AB tiles: GEMM1 + GEMM2 in one launch
    prefetch = swap                      # + the side-stream L2 prefetch of the first weights
    k4 = 1 if swap else 2
    if nblk <= 148 and d % 256 == 0 and E <= 128:  # fused front end: gate + top-k + plan + dispatch
        return 1 + k4 + 1 + prefetch
    tc_gate = T >= 8192 and d % 256 == 0  # tcgen05 gate (+ its side-stream histogram copy to the host)
    split = not tc_gate and nblk * 4 <= 2 * 148  # small batches split K (+ finish kernel)
    # top-2 on the 2-SM kernel: GEMM2 writes y itself (FusedY), no combine launch
    combine = 0 if (not swap and k == 2 and os.environ.get("MOE_FUSED_Y", "1") != "0") else 1
    return 1 + (1 if tc_gate else 0) + split + 1 + 1 + k4 + combine + prefetch


PLANNER = {"sync": "MOE_PLAN_SYNC (scale_experts + place_experts on actual loads)",
           "predicted": "MOE_PLAN_PREDICTED (historical bootstrap planned one step ahead; device-planned forwards)"}


def config_dict(G, c, plan="sync"):
    """The `config` of both arms' lines (identical for the same workload and N)."""
    E, k, d, ff, T = c["E"], c["k"], c["d"], c["ff"], c["T"]
    return {"workload": WORKLOAD, "global_batch": G * T, "tokens_per_gpu": T, "seq_len": None,
            "parallelism": f"ep{G}", "experts": E, "top_k": k, "d_model": d, "d_ff": ff,
            "l2": f"inputs larger than L2 ({E * 3 * d * ff * 2 / 1e9:.2f} GB of expert weights + "
                  f"{T * d * 2 / 1e6:.0f} MB of tokens per step vs 126 MB of L2)",
            "planner": PLANNER[plan]}


def host_cpu():
    """nproc, the threads the CPU path uses, and the CPU model."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "model": model,
            "threads": int(os.environ.get("OMP_NUM_THREADS", "0")) or os.cpu_count()}


# ------------------------------------------------------------ CPU reference path
# Everything below runs the oracle (oracle/_ref = the UNMODIFIED reference's
# planner path, oracle/*.c|py = the restated data path) and never imports the
# product package: the reference arm's process maps only oracle libraries.
def cpu_layer(c, experts=None):
    from oracle import workload as owl
    from oracle.cpu_path import CpuLayer
    E, k, d, ff = c["E"], c["k"], c["d"], c["ff"]
    if experts is None:
        experts = [owl.expert_weights(d, ff, c["seed"], 0, e) for e in range(E)]
    return CpuLayer(E, k, d, ff, experts, s=c["s"], seed=c["seed"], extra_replicas=c["extra_replicas"])


def cpu_sample(c, layer, tokens, it, rank=0):
    """One step of the CPU path on `tokens` tokens of this step's batch (the
    keyed generator makes them a prefix of the full batch) under its gate."""
    from oracle import workload as owl
    x = owl.tokens(tokens, c["d"], c["E"], c["seed"], rank * 1000 + it % 4)
    wg = owl.gate_weights(c["E"], c["d"], c["s"], c["seed"], 0, it)
    _, dt = layer.forward(x, wg)
    return dt


def run_cpu_baseline(c, sample_tokens, experts=None, steps=2):
    layer = cpu_layer(c, experts)
    cpu_sample(c, layer, 64, 0)  # page in
    times = [cpu_sample(c, layer, sample_tokens, i) for i in range(steps)]
    hc = host_cpu()
    return {"value": sample_tokens / statistics.median(times), "unit": "tokens/s", "cores": hc["threads"],
            "kind": "port", "cpu": hc,
            "sample": (f"{sample_tokens} tokens of the {c['T']}-token layer per sample, median of {steps}: the "
                       f"reference's per-layer planner path (oracle/_ref) + the oracle data path (gate, stable "
                       f"dispatch, fp32 SwiGLU FFN on OpenBLAS sgemm, combine) on {hc['threads']} threads "
                       f"({hc['model']})"),
            "ms_per_sample": 1e3 * statistics.median(times)}


def cpu_cfg1_full_layer():
    """The reference's own CPU-runnable configuration (BASELINE.json configs[0],
    cfg1: E8 k2 d1024 ff3584, 2048 tokens) as ONE full layer on the host."""
    c = dict(OTHER_WORKLOADS["cfg1"][0])
    layer = cpu_layer(c)
    cpu_sample(c, layer, 64, 0)
    dt = cpu_sample(c, layer, c["T"], 0)
    hc = host_cpu()
    return {"value": c["T"] / dt, "unit": "tokens/s", "cores": hc["threads"], "kind": "port", "ms_per_layer": 1e3 * dt,
            "sample": "cfg1 in full: one 2048-token layer (E8 k2 d1024 ff3584), reference planner path + oracle "
                      "data path"}


def run_reference(args):
    """--impl reference: the CPU path of this metric on the host's cores, rank 0
    only.  Each step runs a bounded sample of the step's batch (default 4096 of
    16384 tokens: every token's routing and FFN rows are independent, so the
    cost is linear in tokens); one full 16384-token layer is also timed once
    after the steps and reported beside the per-step rate."""
    ws, rank, local = dist_env()
    if rank != 0:
        return 0
    import oracle
    c = CFG
    G = max(ws, 1)
    sample = min(args.cpu_sample_tokens, c["T"])
    layer = cpu_layer(c)
    cpu_sample(c, layer, 64, 0)  # page in the resident fp32 weights
    for i in range(args.warmup):
        cpu_sample(c, layer, sample, i)
    times = [cpu_sample(c, layer, sample, args.warmup + i) for i in range(args.steps)]
    full_s = cpu_sample(c, layer, c["T"], args.warmup + args.steps) if args.cpu_full_layer else None
    total = sum(times)
    value = sample * args.steps / total
    ref = oracle.ref()
    pct = (lambda v, q: ref.ref_percentile((oracle.C.c_double * len(v))(*v), len(v), q)) if ref else None
    ms = [1e3 * t * c["T"] / sample for t in times]  # per-layer latency at the full batch (linear in tokens)
    hc = host_cpu()
    desc = (f"{sample} of the {c['T']} tokens of each step's batch: the UNMODIFIED reference's per-layer "
            f"planner path (oracle/_ref: route_tokens -> predict -> scale_experts -> place_experts -> "
            f"layer_forward_time -> update_registry) + the oracle data path the reference only models "
            f"(gate, stable integer dispatch, fp32 SwiGLU FFN on OpenBLAS sgemm, weighted combine), "
            f"{hc['threads']} threads on {hc['nproc']} x {hc['model']}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (the same keyed inputs as the GPU arm, from the oracle's generator)",
        "config": config_dict(G, c, args.plan),
        "p50_ms": statistics.median(ms), "p99_ms": pct(ms, 0.99) if pct else max(ms),
        "latency_note": "per-layer latency scaled from the sample to the full batch",
        "sample": {"tokens_per_step": sample, "tokens_per_layer": c["T"],
                   "full_layer_s": full_s, "full_layer_tokens_per_s": c["T"] / full_s if full_s else None,
                   "sample_tokens_per_s": value,
                   "extrapolation": "tokens/s of the sample == tokens/s of the layer when the cost is linear "
                                    "in tokens; full_layer_tokens_per_s is the measured check"},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": hc["threads"], "kind": "reference",
                         "cpu": hc, "sample": desc},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "repo_libs_loaded": repo_libs_loaded(),
    }
    assert not any("libmoe_b200" in p for p in line["repo_libs_loaded"]), "reference arm loaded the product"
    print(json.dumps(line), flush=True)
    return 0


def repo_libs_loaded():
    """Shared objects under this repo mapped into the process (/proc/self/maps)."""
    out = set()
    try:
        with open("/proc/self/maps") as f:
            for line in f:
                path = line.split()[-1] if len(line.split()) >= 6 else ""
                if path.startswith(ROOT) and ".so" in path:
                    out.add(os.path.relpath(path, ROOT))
    except OSError:
        pass
    return sorted(out)


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch

    from paper_2603_06350_b200 import (MOE_EXCHANGE_NCCL, MOE_EXCHANGE_P2P, MOE_PLAN_PREDICTED, MOE_PLAN_SYNC,
                                       MoELayer, nccl_unique_id,
                                       percentile)
    from paper_2603_06350_b200 import workload as wl

    ws, rank, local = dist_env()
    G = max(ws, 1)
    # MOE_BENCH_SHARE_DEVICE=1: every rank on device 0 (exercises the N>1 flow on
    # a one-GPU box; the numbers are then not a scaling measurement)
    shared = os.environ.get("MOE_BENCH_SHARE_DEVICE") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if G > 1 and args.exchange == "nccl":
        # communicator lines (nRanks, channels, NVLS) on stderr for the driver's check
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if G > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = CFG
    E, k, d, ff, T = c["E"], c["k"], c["d"], c["ff"], c["T"]
    plan_mode = MOE_PLAN_PREDICTED if args.plan == "predicted" else MOE_PLAN_SYNC
    uid = None
    p2p = G > 1 and args.exchange == "p2p"
    mem = 3.0 * d * ff * 2 / 1e6

    def make_layer(use_p2p):
        uid = None
        if G > 1 and not use_p2p:
            obj = [nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uid = obj[0]
        lay = MoELayer(1, E, k, d, ff, max_tokens=T, world_size=G, rank=rank, device=local,
                       exchange_mode=MOE_EXCHANGE_P2P if use_p2p else MOE_EXCHANGE_NCCL,
                       nccl_unique_id=uid, expert_mem_mb=mem, layer_mem_cap_mb=c["extra_replicas"] * mem,
                       gpu_mem_capacity_mb=180000.0, cv_threshold=0.2, keep_alive_iters=50,
                       residency=1 if (use_p2p and args.residency == "placed") else 0)
        if use_p2p:  # map every rank's exchange slab (CUDA IPC over NVLink)
            handles = [None] * G
            dist.all_gather_object(handles, lay.p2p_export())
            lay.p2p_import(handles)
        for e in range(E):
            lay.load_expert(0, e, *wl.expert_weights(d, ff, c["seed"], 0, e))
        return lay

    exchange_note = None
    if p2p:
        # The peer-memory path is the product; if it cannot be set up on this
        # box (no peer access, IPC refused, a peer out of step) every rank
        # falls back to the NCCL exchange together rather than hanging.
        m, err = None, ""
        try:
            m = make_layer(True)
            m.set_gate(0, wl.gate_weights(E, d, c["s"], c["seed"], 0, 0))
            xt = torch.from_numpy(wl.tokens(T, d, E, c["seed"], rank * 1000).view(np.int16)).cuda()
            m.forward(0, xt, torch.empty_like(xt), MOE_PLAN_SYNC, 0)
            m.sync()
        except Exception as ex:  # noqa: BLE001 - any setup failure selects the fallback
            err = f"{type(ex).__name__}: {ex}"
        ok = torch.tensor([0 if err else 1], dtype=torch.int32, device="cpu" if shared else "cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            print(f"[bench] rank {rank}: peer-memory exchange unavailable ({err or 'a peer failed'}); "
                  "falling back to NCCL", file=sys.stderr, flush=True)
            if m is not None:
                try:
                    m.close()
                except Exception:  # noqa: BLE001
                    pass
            p2p = False
            exchange_note = "NCCL send/recv (peer-memory setup failed: " + (err or "on a peer") + ")"
            m = make_layer(False)
    else:
        m = make_layer(False)
    # token pool: per rank distinct batches (DP shard of the global batch)
    pool_host = [wl.tokens(T, d, E, c["seed"], rank * 1000 + i) for i in range(args.pool)]
    pool = [torch.from_numpy(x.view(np.int16)).cuda() for x in pool_host]
    y = torch.empty((T, d), dtype=torch.int16, device="cuda")
    total_iters = args.warmup + args.steps
    # one gate per iteration (that is what re-routes every step), resident on the
    # device like a model's gate; each step installs its gate with a
    # stream-ordered device copy (moe_set_gate_weights_device)
    gates = torch.from_numpy(np.stack([wl.gate_weights(E, d, c["s"], c["seed"], 0, it)
                                       for it in range(total_iters + args.steps + 2)]).view(np.int16)).cuda()
    stream = torch.cuda.ExternalStream(m.stream_ptr)

    def step(it, stats=True):
        m.set_gate_device(0, gates[it])
        return m.forward(0, pool[it % args.pool], y, plan_mode, it, stats=stats)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    placed = p2p and args.residency == "placed"
    cold = [step(it, stats=placed) for it in range(args.warmup)]  # PLACED: the cold starts happen here
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        t_start.record(stream)
        for i in range(args.steps):
            ev[i][0].record(stream)
            step(args.warmup + i, stats=False)  # no per-step host sync: the host runs ahead
            ev[i][1].record(stream)
        t_end.record(stream)
        barrier()
    total_ms = t_start.elapsed_time(t_end)
    lat = [a.elapsed_time(b) for a, b in ev]
    # K4 times of the TIMED steps: CUDA events the C-ABI records around the two
    # grouped GEMMs of every forward on its stream (no host sync in the loop)
    g1, g2, grows = m.gemm_times(min(args.steps, 64))
    gemm_ms = [float(a + b) for a, b in zip(g1, g2)]
    rows = [int(r) for r in grows]
    # phase breakdown (per-phase events + host sync per call) from a short
    # untimed pass after the timed region
    stats = [step(args.warmup + args.steps + i, stats=True) for i in range(min(args.steps, 10))]
    phases = {name: statistics.median(getattr(s, name) for s in stats)
              for name in ("gate_ms", "plan_ms", "dispatch_ms", "a2a_dispatch_ms", "gemm1_ms", "gemm2_ms",
                           "a2a_combine_ms", "combine_ms")}
    replicas = statistics.median(s.replica_count for s in stats)
    a2a = None
    if G > 1:
        # bytes this rank ships to other ranks per direction; with the peer-memory
        # exchange they move inside dispatch (remote stores) and combine (remote
        # loads), so the bus rate is bounded below by bytes / kernel time
        sent = statistics.median(s.rows_sent for s in stats) * d * 2
        disp = phases["dispatch_ms"] + phases["a2a_dispatch_ms"]
        comb = phases["combine_ms"] + phases["a2a_combine_ms"]
        a2a = {"remote_bytes_per_direction": sent, "dispatch_ms": disp, "combine_ms": comb,
               "bus_gbs_dispatch": sent / (disp * 1e-3) / 1e9 if disp > 0 else None,
               "bus_gbs_combine": sent / (comb * 1e-3) / 1e9 if comb > 0 else None,
               "peak_gbs_per_direction": 900.0,
               "note": "rank 0; dispatch/combine include local rows and the flag handshakes"
                       + ("; ranks share one GPU (not NVLink)" if shared else "")}
    balance = None
    if G > 1:
        # straggler balance of the planner's placement on the same steps: rows
        # each rank's GEMMs ran vs the rows static EP (expert e on GPU e mod G,
        # no replicas; baselines.cpp:32-60) would have put on each rank
        dev = "cpu" if shared else "cuda"
        mine = torch.tensor([[float(s.rows_local) for s in stats]], dtype=torch.float64, device=dev)
        allr = [torch.zeros_like(mine) for _ in range(G)]
        dist.all_gather(allr, mine)
        per_rank = torch.cat(allr).cpu().numpy()                       # [G, steps]
        cnt = torch.tensor([[float(v) for v in s.counts[:E]] for s in stats], dtype=torch.float64, device=dev)
        dist.all_reduce(cnt)                                            # global histogram per step
        cnt = cnt.cpu().numpy()
        static = np.stack([cnt[:, [e for e in range(E) if e % G == g]].sum(axis=1) for g in range(G)])
        ratio = lambda a: float(np.median(a.max(axis=0) / np.maximum(a.mean(axis=0), 1.0)))
        # oracle_balance_time (baselines.cpp:141-154): the GEMM time every rank
        # would need with the rows spread perfectly, from rank 0's per-row rate
        rows0 = statistics.median(s.rows_local for s in stats)
        gemm0 = statistics.median(s.gemm1_ms + s.gemm2_ms for s in stats)
        balance = {"rows_per_rank_median": [float(v) for v in np.median(per_rank, axis=1)],
                   "max_over_mean": ratio(per_rank), "static_ep_max_over_mean": ratio(static),
                   "gemm_ms_perfect_balance": gemm0 / max(rows0, 1) * float(np.median(per_rank.mean(axis=0))),
                   "gemm_ms_slowest_rank_est": gemm0 / max(rows0, 1) * float(np.median(per_rank.max(axis=0))),
                   "note": "median over the stats steps; 1.0 = perfectly balanced ranks; GEMM ms from rank 0's "
                           "per-row rate (the oracle_balance_time line)"}
    residency = None
    if p2p and args.residency == "placed":
        residency = {"mode": "placed (home experts + replica cache slots, cold copies from the home GPU)",
                     "copies_per_step": statistics.mean(s.weight_copies for s in stats),
                     "hits_per_step": statistics.mean(s.weight_hits for s in stats),
                     "copy_ms_median_when_cold": statistics.median(
                         [s.weight_copy_ms for s in stats if s.weight_copies] or [0.0]),
                     "copy_mb_per_step": statistics.mean(s.weight_copy_mb for s in stats),
                     "warmup_copies": [s.weight_copies for s in cold],
                     "warmup_copy_ms": [round(s.weight_copy_ms, 3) for s in cold],
                     "warmup_forward_ms": [round(s.forward_ms, 3) for s in cold],
                     "note": "copy time measured on the weight stream (peer copy engine); with "
                             "MOE_BENCH_SHARE_DEVICE the 'peer' is the same GPU (D2D, not NVLink)"}

    # e2e through the host-buffer C-ABI entry point
    e2e = None
    if not args.no_e2e:
        # pinned host batches in, pinned host outputs out, pipelined C-ABI calls
        xh = [torch.from_numpy(x.view(np.int16)).pin_memory() for x in pool_host]
        yh = [torch.empty((T, d), dtype=torch.int16).pin_memory() for _ in range(3)]
        tickets = []
        for i in range(2):  # warm the staging buffers / streams
            m.set_gate_device(0, gates[i])
            tickets.append(m.forward_host_async(0, xh[i % len(xh)], yh[i % 3], plan_mode, i))
        for t in tickets:
            m.wait(t)
        barrier()
        tickets = []
        t0 = time.perf_counter()
        for i in range(args.steps):
            it = total_iters + i
            if i >= 3:
                m.wait(tickets[i - 3])  # its output buffer is about to be reused
            m.set_gate_device(0, gates[it])
            tickets.append(m.forward_host_async(0, xh[i % len(xh)], yh[i % 3], plan_mode, it))
        for t in tickets[-3:]:
            m.wait(t)
        e2e_ms = (time.perf_counter() - t0) * 1e3  # host-visible: every result is in host memory
        barrier()
        e2e = {"ms": e2e_ms}

    # max over ranks
    vals = torch.tensor([total_ms, statistics.median(lat), nearest_rank(lat, 0.99),
                         e2e["ms"] if e2e else 0.0], dtype=torch.float64, device="cpu" if shared else "cuda")
    if dist is not None:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    total_ms, p50, p99, e2e_ms = vals.tolist()

    if rank == 0:
        peaks, peak_src = load_peaks()
        gflop = [2.0 * r * d * 2 * ff + 2.0 * r * ff * d for r in rows]
        achieved = statistics.median(f / (t * 1e-3) / 1e12 for f, t in zip(gflop, gemm_ms))
        # the burst figure for a kernel timed in a short region (the driver's 20 steps
        # are ~0.16 s), the power-capped sustained one for seconds-long runs
        long_run = total_ms > 1000.0
        peak_kind = "sustained" if long_run else "burst"
        peak = (peaks.get("bf16_tflops_sustained") if long_run else None) or peaks.get("bf16_tflops")
        traffic = ncu_traffic()
        line = {
            "metric": METRIC,
            "value": G * T * args.steps / (total_ms * 1e-3),
            "unit": "tokens/s",
            "n_gpus": G, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (keyed Zipf-skewed gate inputs, random-init expert weights)",
            "config": config_dict(G, c, args.plan),
            "exchange": (exchange_note or ("peer memory (P2P)" if p2p else "NCCL send/recv")) if G > 1
                        else "none (G=1)",
            "p50_ms": p50, "p99_ms": p99,
            "step_ms": [round(v, 3) for v in lat],
            "phase_ms_median": phases, "replicas_median": replicas,
            # our kernels per step.  G=1: K1 gate (+ its split-K finish for small
            # batches; it also mirrors the histograms to the host), block prefix + on-device
            # plan (one launch; folded into dispatch for <= 32 token blocks), K3 dispatch,
            # K4 GEMM1 + GEMM2 (one launch for the swap-AB tiles of small batches), K5 combine.
            # P2P (host-planned SYNC steps): gate, counts gather, counts SM copy, plan upload,
            # prefix, dispatch, rows wait, GEMM1, GEMM2, outputs signal + wait, combine.  NCCL:
            # gate, counts copy, plan upload, prefix, dispatch, GEMM1, GEMM2, combine (NCCL's own
            # kernels and the gate-weight memcpy not counted)
            "gpu_launches": (12 if p2p else (8 if G > 1 else single_gpu_launches(T, k, E, d))) * args.steps,
            "roofline": {"bound": "tensor", "kernel": "grouped_gemm_2sm_kernel (GEMM1 SwiGLU + GEMM2)",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                         "peak_source": f"{peak_src}, bf16 {peak_kind} (timed region {total_ms / 1e3:.2f} s)",
                         "burst_peak": peaks.get("bf16_tflops"),
                         "sustained_peak": peaks.get("bf16_tflops_sustained"),
                         "algorithmic_flops_per_step": statistics.median(gflop),
                         "kernel_ms_per_step": statistics.median(gemm_ms),
                         "timing": "CUDA events around GEMM1/GEMM2 of each timed step on the ctx stream "
                                   "(moe_gemm_times); achieved = 6*d*ff*rows / (GEMM1+GEMM2), median over steps",
                         "traffic": (traffic or {}).get("dram_bytes_per_step"),
                         "traffic_source": (traffic or {}).get("source")},
            "clocks": clk.summary(),
        }
        clk_sum = line["clocks"]
        if clk_sum.get("energy_j"):
            # the K4 clock is set by the board power cap: energy per step is the
            # figure a faster kernel has to lower
            jps = clk_sum["energy_j"] / args.steps
            line["energy"] = {"joules_per_step": jps, "avg_power_w": clk_sum["energy_j"] / (total_ms * 1e-3),
                              "power_limit_w": clk_sum.get("power_limit_w"),
                              "k4_tflop_per_joule": statistics.median(gflop) / jps / 1e12,
                              "note": "whole board, timed region (includes the counter's sampling slack)"}
        if residency is not None:
            line["residency"] = residency
        if a2a is not None:
            line["all_to_all"] = a2a
        if balance is not None:
            line["straggler_balance"] = balance
        if e2e is not None:
            xb = T * d * 2
            line["e2e"] = {"value": G * T * args.steps / (e2e_ms * 1e-3), "unit": "tokens/s",
                           "h2d_bytes_per_step": xb, "d2h_bytes_per_step": T * d * 2,
                           "ms_per_step": e2e_ms / args.steps,
                           "api": "moe_layer_forward_host_async + moe_wait (C-ABI, pinned host buffers; "
                                  "H2D/D2H of neighbouring steps overlap the layer), wall clock over all steps "
                                  "until the last result is in host memory"}
        if G == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = run_cpu_baseline(c, args.cpu_baseline_tokens,
                                                    [wl.expert_weights(d, ff, c["seed"], 0, e) for e in range(E)])
            line["cpu_baseline_cfg1_full"] = cpu_cfg1_full_layer()
        print(json.dumps(line), flush=True)
    m.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    global CFG, WORKLOAD
    args = parse()
    if args.plan is None:
        args.plan = "predicted" if int(os.environ.get("WORLD_SIZE", "1")) > 1 else "sync"
    if args.workload != "cfg2":
        CFG, WORKLOAD = OTHER_WORKLOADS[args.workload]
    if args.impl == "reference":
        # all host threads for the CPU path: torchrun (N > 1) exports OMP_NUM_THREADS=1 to every
        # rank, and only rank 0 runs this arm; set before numpy / OpenBLAS / the oracle load
        threads = os.environ.get("MOE_REF_THREADS") or str(os.cpu_count() or 1)
        for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS"):
            os.environ[var] = threads
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
