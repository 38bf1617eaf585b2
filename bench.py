"""Headline benchmark: served requests/s and on-time ratio of live batch-aware
serving on B200 (BASELINE.json metric; config 2 of its configs).

Workload (config 2): GoogLeNet 224x224 single DNN, Poisson arrivals, the
on-time-ratio objective (Our-Tardy DP, reference deadline.hpp:130-282) with
partial batching at layer granularity, B = 90, on 1 B200 (N GPUs: one
independent server per GPU, weak scaling, no collectives on the data path).
The scheduler plans on the latency table h_k(b) MEASURED at startup on this
GPU (reference profile schema, after the profile-time launch autotune); the
deadline is D = 6.25 x T1 with T1 the single-request latency
of the committed B200 table of the config (profiles/r02/*_table_b200.json,
measured by this executor at the start of round 2), so the SLO is fixed and
the reference arm serves the same deadline; the capacity at 6.25 x today's
T1 is reported beside it ("capacity_at_current_t1_deadline").

A "step" is one live serving run of R requests arriving as a Poisson stream
at the offered rate lambda*, where lambda* is the measured capacity (largest
rate with on-time ratio >= 0.90, reference simulator.hpp:804-820), found by
the warm-up runs. value = requests completed / device time of the K timed
runs (CUDA events on the serving stream), summed over ranks / max over ranks.
Inputs are synthetic images resident in HBM for `value`; `e2e` repeats the
timed runs through the public C-ABI with each request's image copied H2D
from pinned host memory at admission and its class probabilities copied
D2H at completion.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "served requests/s (Poisson, on-time >= 0.90 capacity point), GoogLeNet config 2"
UNIT = "req/s"
BATCHES = (1, 2, 4, 8, 12, 16, 24, 32, 48, 64, 90)


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        # BENCH_ONE_DEVICE=1 + BENCH_DIST_BACKEND=gloo: every rank on GPU 0, a
        # functional check of the N > 1 path on a one-GPU box (its timings
        # mean nothing: the ranks share one GPU).
        if os.environ.get("BENCH_ONE_DEVICE") == "1":
            local = 0
        torch.cuda.set_device(local)
        dist.init_process_group(_backend(), init_method="env://")
    return ws, rank, local


def _backend() -> str:
    return os.environ.get("BENCH_DIST_BACKEND", "nccl")


def _red_device() -> str:
    return "cpu" if _backend() == "gloo" else "cuda"


def allreduce_max(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=_red_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=_red_device())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(ws: int):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def peaks() -> dict:
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        p.update({k: d[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in d})
        p["source"] = "MEASURED_PEAKS.json"
    # TF32 dense tensor rate is half the bf16 rate on Blackwell (2.25 vs 1.1
    # PFLOP/s nominal); derive it from the measured sustained bf16 figure.
    p["tf32_tflops"] = p["bf16_tflops_sustained"] / 2.0
    return p


class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = Path("/tmp") / f"bs_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.QUERY}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in self.path.read_text().splitlines():
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9:
                    continue
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
                for n, v in zip(names, f[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
        except Exception:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# BASELINE.json configs measured live (config 5, collaborative offload, runs
# in replay only: its client side is modelled, tests/test_executor_gpu.py).
CONFIGS = {
    1: {"suite": "small_cnn", "max_batch": 10, "deadline_ms": 0.569, "process": "constant", "scheduler": "ours-time",
        "granularity": "request",
        "workload": "config 1: SmallCNN 32x32 single DNN, Constant arrivals, completion-time DP (Ours-Time), "
                    "request granularity, B=10"},
    2: {"suite": "googlenet", "max_batch": 90, "deadline_ms": 3.559, "process": "poisson", "scheduler": "ours-tardy",
        "granularity": "layer",
        "workload": "config 2: GoogLeNet 224x224 single DNN, Poisson arrivals, Our-Tardy (on-time objective), "
                    "partial batching at layer granularity, B=90, 1 server per GPU"},
    3: {"suite": "resnet50_pair", "max_batch": 90, "deadline_ms": 7.072, "process": "pareto", "scheduler": "ours-time",
        "granularity": "group", "shared_batching": True, "depth": 2,  # Pareto bursts: 2 in flight +4% (profiles/r02/serving_steps/depth_c3_sparse_sampling.txt)
        "workload": "config 3: two DNNs sharing a ResNet-50 backbone (heads 1000 / 365 classes), shared-layer "
                    "merge batching with riders, Pareto arrivals (alpha 1.25), G=5, B=90"},
    4: {"suite": "hetero3", "max_batch": 90, "deadline_ms": 6.949, "process": "poisson", "scheduler": "ours-time",
        "granularity": "group",
        "workload": "config 4: GoogLeNet + ResNet-50 + MobileNetV2 (no shared layers), equal Poisson mix, "
                    "multi-DNN permutation DP, G=5, B=90, request streams sharded over GPUs"},
    5: {"suite": "collab", "max_batch": 90, "deadline_ms": 11.226, "process": "pareto", "scheduler": "ours-tardy",
        "granularity": "group", "offload": "partial", "clients": 1024, "deadline_t1_factor": 12.5,
        "workload": "config 5: collaborative partial offload (GoogLeNet + ResNet-50, Jetson Nano client "
                    "profile, LTE uplink trace x10, 1024 clients, request -> client (id - 1) % clients); the "
                    "client side replayed by the reference-semantics simulator, the server suffixes served "
                    "live; congested Pareto arrivals, Our-Tardy, G=5, B=90, D = 12.5 x T1 (the paper's "
                    "300 ms collaborative deadline = 2 x 150 ms)"},
}


def run_ours(a, ws, rank, local) -> dict | None:
    from paper_2304_09961_b200.executor import Executor

    cfg = CONFIGS[a.config]
    pk = peaks()
    mb = cfg["max_batch"]
    # Programmatic dependent launch is on by default (a config may opt out
    # with "pdl": False; none does since the latency tables are scaled to the
    # whole-pass time, pdl.cuh). An explicit BS_PDL in the environment wins.
    # Read once, before the first launch.
    if not cfg.get("pdl", True):
        os.environ.setdefault("BS_PDL", "0")
    pdl_on = os.environ.get("BS_PDL", "1") != "0"
    ex = Executor(cfg["suite"], device=local, max_batch=mb, max_requests=a.slots)
    ex.set_precision(a.precision)
    # The executor first autotunes each N > 128 conv's tile width per batch
    # (kept for the run), then measures the latency table the scheduler uses.
    prof = ex.profile_table(batches=[b for b in BATCHES if b < mb] + [mb], reps=10, tune_tiles=True,
                            flush_l2=a.table_flush_l2, timing=table_timing(cfg))
    prof.pop("tile_tune", None)
    names = [n["name"] for n in ex.desc["nets"]]
    comp = {c["id"]: c for c in prof["components"]}

    def dnn_ms(d, b):
        return sum(dict(L["runtime_ms"])[b] for cid in d["stages"] for L in comp[cid]["layers"])

    # Every rank measures its own table (independent servers), but the rates
    # probed must be the same on every rank (one global trace, sharded): start
    # the capacity search from the slowest rank's table.
    t1 = allreduce_max(max(dnn_ms(d, 1) for d in prof["dnns"]), ws)
    tmax = allreduce_max(max(dnn_ms(d, mb) for d in prof["dnns"]), ws)
    # D = 6.25 x T1 (the paper's 150 ms / 24 ms ratio), T1 =
    # the single-request latency of the slowest DNN in the committed B200
    # table of this config (profiles/r02, measured by this executor; the
    # reference arm simulates on the same table, so both arms serve the same
    # deadline); the fresh startup table's T1 is reported beside it and used
    # when no table is committed. --deadline-ms overrides (reported).
    # The workload's deadline is fixed per config (CONFIGS deadline_ms: 6.25 x
    # T1 -- 12.5 x for config 5 -- of the B200 tables committed at the start
    # of round 2, per-layer event timings), so both arms and every run serve
    # the same D however T1 evolves; --deadline-ms overrides (reported).
    t1_table = committed_t1(a.config)
    factor = cfg.get("deadline_t1_factor", 6.25)
    deadline = a.deadline_ms if a.deadline_ms else cfg["deadline_ms"]
    sim = sim_config(cfg, mb)
    depth = int(os.environ.get("BENCH_DEPTH", cfg.get("depth", 4)))  # env: A/B
    # steps in flight in the live loop: 4. With the pass-scaled tables 3 beat 2
    # (config 2 +5%, 4 +11%, 5 +6%, 1 +3%, 3 -4% within noise;
    # profiles/r02/depth/); with the serving-step chain (pointer-table kernel,
    # reference admission) config 2 at 57k offered is on time 0.90 at 4 vs
    # 0.83-0.87 at 3 and 0.81-0.86 at 6, 0.75-0.81 at 8 (deeper plans further
    # ahead of the arrivals), configs 1 / 3 / 4 neutral
    # (profiles/r02/serving_steps/depth_*.txt)
    # Planning margin (A/B switch, default 1.0 = plan on the measured table):
    # every h_k(b) the scheduler sees is scaled by it.
    margin = float(os.environ.get("BENCH_TABLE_MARGIN", cfg.get("table_margin", 1.0)))
    plan_prof = prof
    if margin != 1.0:
        import copy
        plan_prof = copy.deepcopy(prof)
        for c in plan_prof["components"]:
            for L in c["layers"]:
                L["runtime_ms"] = [[b, ms * margin] for b, ms in L["runtime_ms"]]
    base = dict(collab_inputs(cfg), profile=plan_prof, sim=sim, image_pool=64, pipeline_depth=depth)

    def job(rate, count, seed, h2d=False, dl=None):
        """One serving run. N > 1: ONE global trace (N x the per-GPU rate and
        count, the same seed on every rank) routed round-robin by request id
        (paper_2304_09961_b200/shard.py); each rank serves its shard as
        explicit arrivals, so every shard is replayable through the reference
        simulator for per-shard schedule parity."""
        w = {"process": cfg["process"], "rate": rate * ws, "count": count * ws, "seed": seed,
             "relative_deadline": dl or deadline}
        if len(names) > 1:
            w["dnn_mix"] = [[n, 1.0 / len(names)] for n in names]
        j = dict(base, workload=w, h2d=h2d)
        if ws > 1:
            from paper_2304_09961_b200.shard import shard_job
            j = shard_job(j, ws, rank)[0]
        return j
    t90 = tmax

    # ---- warm-up: capacity search (largest offered rate per GPU with the
    # whole job's on-time ratio >= 0.9; the same decisions on every rank)
    def serve_trial(rate, i):
        # three traces per probed rate: near saturation the on-time ratio of a
        # single 3000-request trace varies by +-0.05 from seed to seed
        on = gen = 0
        for s in range(3):
            r = ex.serve(job(rate, a.warm_requests, 1000 + 10 * i + s))
            on += r["on_time"]
            gen += r["generated"]
        return allreduce_sum(on, ws) / max(1.0, allreduce_sum(gen, ws))

    cap_search, warm_runs = capacity_search(serve_trial, mb / t90 * 1000.0, a.warmup)
    # Timed runs at 97% of the largest passing rate: the on-time ratio is steep
    # near saturation and single runs vary by a few percent.
    cap = cap_search * 0.97

    # ---- timed steps at the capacity rate. The timed region must itself meet
    # the 0.90 on-time bar (the capacity definition); if it does not, the
    # rate is lowered (step_down: 4% near the bar) and the K steps are timed
    # again (at most six times).
    retimed = []
    for attempt in range(7):
        ex.stats(True, every=a.stats_every)
        completed = generated = on_time = launches = 0
        device_ms = 0.0
        sched = []
        with ClockSampler(local) as clk:
            barrier(ws)
            t_wall = time.perf_counter()
            # BENCH_PROFILE_TIMED=1: profiler range around the timed steps only,
            # for `ncu --profile-from-start off` launch lists of the timed region
            if os.environ.get("BENCH_PROFILE_TIMED") == "1" and attempt == 0:
                import ctypes
                ctypes.CDLL("libcudart.so.12").cudaProfilerStart()
            for k in range(a.steps):
                r = ex.serve(job(cap, a.requests, 5000 + k))
                completed += r["completed"]
                generated += r["generated"]
                on_time += r["on_time"]
                launches += r["launches"]
                device_ms += r["device_ms"]
                sched.append(r)
            barrier(ws)
            wall_ms = (time.perf_counter() - t_wall) * 1000
            if os.environ.get("BENCH_PROFILE_TIMED") == "1" and attempt == 0:
                import ctypes
                ctypes.CDLL("libcudart.so.12").cudaProfilerStop()
        ratio = allreduce_sum(on_time, ws) / max(1.0, allreduce_sum(generated, ws))
        if ratio >= 0.90 or attempt == 6:
            break
        retimed.append([round(cap, 1), round(ratio, 4)])
        ex.stats(False)
        cap = step_down(cap, ratio)
    clocks = clk.summary()
    # tensor peak of the arithmetic this run uses (BF16: the measured bf16 rate)
    tc_peak = pk["bf16_tflops_sustained"] if a.precision == "bf16" else pk["tf32_tflops"]
    stats = ex.stats_summary(pk["hbm_gbs"], tc_peak)
    ex.stats(False)

    # ---- e2e: same runs through the C-ABI with H2D inputs / D2H results.
    # Same metric: served req/s at a rate where the on-time ratio still meets
    # 0.90. Starts at the device-resident rate and steps down (step_down) when
    # the H2D admission path cannot hold the deadlines there.
    def e2e_run(rate):
        c = on = gen = hb = db = 0
        ms = 0.0
        barrier(ws)
        for k in range(a.steps):
            r = ex.serve(job(rate, a.requests, 5000 + k, h2d=True))
            c += r["completed"]
            on += r["on_time"]
            gen += r["generated"]
            ms += r["device_ms"]
            hb += r["h2d_bytes"]
            db += r["d2h_bytes"]
        barrier(ws)
        return {"rate": rate, "completed": c, "ms": ms, "h2d": hb, "d2h": db,
                "ratio": allreduce_sum(on, ws) / max(1.0, allreduce_sum(gen, ws))}

    e2e_cap = cap
    e2e_steps_down = []
    for attempt in range(7):
        run = e2e_run(e2e_cap)
        if run["ratio"] >= 0.90 or attempt == 6:
            break
        e2e_steps_down.append([round(e2e_cap, 1), round(run["ratio"], 4)])
        e2e_cap = step_down(e2e_cap, run["ratio"])
    # After a coarse step-down (15% / 30%) the capacity lies between the last
    # failing and the passing rate: up to three bisections, keeping the
    # highest passing rate's runs (the same capacity rule as the device path).
    if e2e_steps_down and run["ratio"] >= 0.90:
        lo, hi = e2e_cap, e2e_steps_down[-1][0]
        for _ in range(3):
            if hi / lo < 1.04:
                break
            mid = (lo * hi) ** 0.5
            trial = e2e_run(mid)
            if trial["ratio"] >= 0.90:
                run, lo = trial, mid
            else:
                e2e_steps_down.append([round(mid, 1), round(trial["ratio"], 4)])
                hi = mid
        e2e_cap = run["rate"]
    e2e_completed, e2e_ms, h2d, d2h, e2e_ratio = run["completed"], run["ms"], run["h2d"], run["d2h"], run["ratio"]

    # The deadline rule applied to today's executor: D = 6.25 x T1 of the
    # startup table (tighter as single-request latency improves). Capacity
    # search only (reported beside the headline, which keeps the committed
    # table's deadline shared with the reference arm).
    d_now = round(factor * t1, 3)
    at_current_t1 = None
    if not a.deadline_ms and abs(d_now - deadline) > 1e-3:
        def serve_now(rate, i):
            r = ex.serve(job(rate, a.warm_requests, 3000 + i, dl=d_now))
            return allreduce_sum(r["on_time"], ws) / max(1.0, allreduce_sum(r["generated"], ws))
        cap_now, runs_now = capacity_search(serve_now, mb / t90 * 1000.0, a.warmup)
        at_current_t1 = {"deadline_ms": d_now, "t1_ms": round(t1, 4), "capacity_search_rate": round(cap_now, 1),
                         "capacity_search": [[round(r, 1), round(x, 4)] for r, x in runs_now]}

    tot_completed = allreduce_sum(completed, ws)
    tot_gen = allreduce_sum(generated, ws)
    tot_on = allreduce_sum(on_time, ws)
    t_max = allreduce_max(device_ms, ws)
    e2e_tot = allreduce_sum(e2e_completed, ws)
    e2e_t = allreduce_max(e2e_ms, ws)

    conv = stats.get("conv_tc", {})
    roof = None
    if conv:
        tensor_bound = conv["ideal_tensor_ms"] >= conv["ideal_hbm_ms"]
        if tensor_bound:
            ach = conv["flops"] / (conv["ms"] * 1e-3) / 1e12
            roof = {"bound": "tensor", "achieved": round(ach, 2), "peak": tc_peak, "unit": "TFLOP/s"}
        else:
            ach = conv["bytes"] / (conv["ms"] * 1e-3) / 1e9
            roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": pk["hbm_gbs"], "unit": "GB/s"}
        roof["frac"] = round(roof["achieved"] / roof["peak"], 4)
        roof["frac_of_roofline_mixed"] = round(conv["ideal_ms"] / conv["ms"], 4)
        roof["kernel"] = {"tf32x2": "conv_tc_kernel (tcgen05 TF32 implicit GEMM, 2xTF32 split-A)",
                          "tf32": "conv_tc_kernel (tcgen05 TF32 implicit GEMM)",
                          "bf16": "conv_tc_kernel (tcgen05 kind::f16 BF16 implicit GEMM)"}[a.precision]
        roof["sampled_launches"] = conv["launches"]
        roof["avg_launch_us"] = round(conv["ms"] / conv["launches"] * 1000, 2)
        roof["peak_source"] = (f"{pk['source']}: " + ("bf16_tflops_sustained" if a.precision == "bf16" else
                               "tf32 = bf16_tflops_sustained / 2") + "; hbm_gbs measured copy")
        # DRAM bytes per launch: ncu's dram read + write over every conv_tc launch
        # of the config-2 workload replayed at capacity, as a ratio to the
        # algorithmic bytes of the same launches (profiles/ncu_conv_summary.json),
        # applied to this run's algorithmic bytes per launch (the launch mixes
        # differ; the ratio is the comparable figure). < 1: activations written
        # by one layer are read from L2 by the next.
        tr = ncu_traffic()
        alg_per_launch = conv["bytes"] / conv["launches"]
        roof["traffic"] = round(tr * alg_per_launch, 1) if tr is not None else None
        roof["traffic_over_algorithmic"] = round(tr, 4) if tr is not None else None
        roof["algorithmic_bytes_per_launch"] = round(alg_per_launch, 1)
        # The TF32 MMA rate measured on this part (profiles/r01/micro_b200.txt,
        # tools/micro/mma_micro.cu: one 128x128x8 MMA per 64 cycles per SM) at
        # the SM clock sampled during the run. 2xTF32 issues two MMAs per
        # algorithmic MAC, so tensor_pipe_frac = 2 * achieved / this rate;
        # BF16 MMAs run at twice the TF32 rate, one per MAC.
        import torch
        sms = torch.cuda.get_device_properties(0).multi_processor_count
        mhz = (clocks or {}).get("sm_mhz") or 1965.0
        mma_rate = 2 * 128 * 128 * 8 / 64 * sms * mhz * 1e6 / 1e12
        roof["tf32_mma_rate_measured"] = round(mma_rate, 1)
        passes_per_rate = {"tf32x2": 2.0, "tf32": 1.0, "bf16": 0.5}[a.precision]
        roof["tensor_pipe_frac"] = round(passes_per_rate * ach / mma_rate, 4) if tensor_bound else None
        total_ms = sum(v["ms"] for v in stats.values())
        roof["share_of_device_time"] = round(conv["ms"] / total_ms, 4) if total_ms else None

    if rank != 0:
        return None
    out = {
        "metric": METRIC if a.config == 2 else
        f"served requests/s ({cfg['process']}, on-time >= 0.90 capacity point), config {a.config}",
        "value": round(tot_completed / (t_max / 1000.0), 2) if t_max else 0.0,
        "unit": UNIT,
        "n_gpus": ws,
        "steps": a.steps,
        "warmup": a.warmup,
        "ms_per_step": round(t_max / a.steps, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": {"tf32x2": "f32 (tf32x2 tcgen05 MMA, fp32 accumulate)", "tf32": "f32 (tf32 MMA)",
                  "bf16": "bf16 (bf16 tcgen05 MMA operands, fp32 accumulate, fp32 activations)"}[a.precision],
        "data": "synthetic 8-bit RGB images (SplitMix64 N(0,1) draws quantised to 1/32 steps; e2e ships the "
                "bytes, the device path holds their exact fp32 values), deterministic calibrated random-init weights",
        "on_time_ratio": round(tot_on / tot_gen, 4) if tot_gen else None,
        "config": {
            "workload": cfg["workload"],
            "suite": cfg["suite"],
            "offered_rate_per_gpu": round(cap, 1),
            "capacity_search_rate": round(cap_search, 1),
            "requests_per_step": a.requests,
            "deadline_ms": round(deadline, 4),
            "t1_ms": round(t1, 4),
            "t1_ms_committed_table": round(t1_table, 4) if t1_table else None,
            "deadline_rule": "override" if a.deadline_ms else
                             f"fixed per config: {factor} x T1 of the B200 tables committed at the start of round 2 "
                             "(capacity at the same rule on today's T1: capacity_at_current_t1_deadline)",
            "t_max_batch_ms": round(t90, 4),
            "max_batch": mb,
            "precision": a.precision,
            "pdl": pdl_on,
            "pipeline_depth": int(os.environ.get("BENCH_DEPTH", cfg.get("depth", 4))),
            "table_margin": margin,
            "latency_table": "cold L2 (flushed before every timed layer)" if a.table_flush_l2 else
                             f"warm L2, timing '{table_timing(cfg)}' (median of back-to-back repetitions)",
            "l2": "no flush: each step touches R x 4.6 MB request blobs (>> 126 MB L2) plus 26 MB of weights",
            "parallelism": f"{ws} independent servers (request streams sharded, no collectives)",
        },
        "capacity_search": [[round(r, 1), round(x, 4)] for r, x in warm_runs],
        "capacity_at_current_t1_deadline": at_current_t1,
        "retimed_below_target": retimed,
        "latency_ms": {"mean": round(statistics.mean(s["mean_completion_ms"] for s in sched), 4),
                       "p95": round(max(s["p95_completion_ms"] for s in sched), 4)},
        "scheduler_ms": {"mean_per_plan": round(sum(s["sched_ms_total"] for s in sched) /
                                                max(1, sum(s["plans"] for s in sched)), 4),
                         "max": round(max(s["sched_ms_max"] for s in sched), 4)},
        "e2e": {"value": round(e2e_tot / (e2e_t / 1000.0), 2) if e2e_t else 0.0, "unit": UNIT,
                "offered_rate_per_gpu": round(e2e_cap, 1), "on_time_ratio": round(e2e_ratio, 4),
                "stepped_down_from": e2e_steps_down,
                "h2d_bytes_per_step": h2d // max(1, a.steps), "d2h_bytes_per_step": d2h // max(1, a.steps)},
        "gpu_launches": launches,
        "clocks": clocks,
        "roofline": roof,
        "kernel_stats": stats,
        "wall_ms_timed": round(wall_ms, 1),
    }
    out["layer_rooflines"] = layer_rooflines(ex.desc, prof, pk, tc_peak=tc_peak,
                                             w_bytes=2.0 if a.precision == "bf16" else 4.0) if len(names) == 1 else None
    if a.dump_table:
        Path(a.dump_table).parent.mkdir(parents=True, exist_ok=True)
        Path(a.dump_table).write_text(json.dumps(dict(prof, _meta={
            "measured": "bench.py startup on one B200 (per-layer events inside back-to-back passes scaled to the whole-pass time, median of 10)",
            "precision": a.precision, "suite": cfg["suite"]}), indent=1))
    try:
        # rank 0 at N = 1 only (at N > 1 the reference arm's own run carries it)
        out["cpu_baseline"] = (reference_baseline(job(cap, a.requests, 0), cap, 2, 5000) if ws == 1 else
                               {"unavailable": "reported at N = 1 only"})
    except Exception as e:  # the oracle binary is built where the reference is mounted
        out["cpu_baseline"] = {"unavailable": str(e)[:200]}
    out["cpu_forward_img_s"] = cpu_forward(cfg["suite"]) if (a.config == 2 and a.cpu_forward and ws == 1) else None
    return out


def ncu_traffic():
    """DRAM bytes / algorithmic bytes of conv_tc launches from the committed ncu
    launch list (tools/traffic_replay.py, tools/traffic_summary.py)."""
    f = ROOT / "profiles" / "ncu_conv_summary.json"
    if f.exists():
        try:
            return json.loads(f.read_text()).get("dram_over_algorithmic")
        except Exception:
            return None
    return None


REF_DUMP = ROOT / "oracle" / "_ref" / "ref_dump"
TABLES = {1: ROOT / "profiles" / "r02" / "small_cnn_table_b200.json",
          2: ROOT / "profiles" / "r02" / "googlenet_table_b200.json",
          3: ROOT / "profiles" / "r02" / "resnet50_pair_table_b200.json",
          4: ROOT / "profiles" / "r02" / "hetero3_table_b200.json",
          5: ROOT / "profiles" / "r02" / "collab_table_b200.json"}


def sim_config(cfg: dict, mb: int) -> dict:
    sim = {"scheduler": cfg["scheduler"], "granularity": cfg["granularity"], "max_batch": mb}
    for k in ("shared_batching", "offload", "clients"):
        if k in cfg:
            sim[k] = cfg[k]
    return sim


def collab_inputs(cfg: dict) -> dict:
    """Client profile and uplink trace of the collaborative config (the
    reference's data files, tests/golden/ref_data)."""
    if "offload" not in cfg:
        return {}
    data = ROOT / "tests" / "golden" / "ref_data"
    return {"client_profile": str(data / "jetson_nano.json"), "trace": str(data / "lte_uplink.csv"),
            "trace_scale": 10.0}


def committed_t1(config: int) -> float | None:
    """T1 (single-request latency, slowest DNN) of the committed B200 table."""
    table = TABLES.get(config)
    if table is None or not table.exists():
        return None
    prof = json.loads(table.read_text())
    comp = {c["id"]: c for c in prof["components"]}
    return max(sum(dict(L["runtime_ms"])[1] for cid in d["stages"] for L in comp[cid]["layers"])
               for d in prof["dnns"])


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def ref_runs(job: dict, runs: list[dict]) -> list[dict]:
    """The reference's run_sim (oracle/_ref/ref_dump, compiled unmodified from
    proj/include/batchsim) on one host core (taskset -c 0): one result line
    per (rate, seed) run — outcome summary, served req/s in simulated time,
    host wall time."""
    if not REF_DUMP.exists():
        raise FileNotFoundError(f"{REF_DUMP} missing (build() compiles it where /root/reference is mounted)")
    cmd = [str(REF_DUMP), "-"]
    if subprocess.run(["which", "taskset"], capture_output=True).returncode == 0:
        cmd = ["taskset", "-c", "0"] + cmd
    r = subprocess.run(cmd, input=json.dumps(dict(job, job="bench", runs=runs)), capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"ref_dump failed: {r.stderr[-400:]}")
    return [json.loads(x) for x in r.stdout.splitlines() if x.strip()]


def table_timing(cfg: dict) -> str:
    """How the startup latency table is timed (Executor.profile_table): layer
    granularity serves one-layer steps, so each layer is timed as such a step
    ("step"); the group / request granularities serve multi-layer steps, whose
    layers overlap inside the launch chain as in a whole pass ("pass": layers
    inside back-to-back passes, scaled to the pass). Measured: config 2 serves
    more on the step table (depth 4: 57k offered on time 0.90 vs 0.83-0.87
    earlier), config 4 on the pass table (11k offered: 1.00 vs 0.87;
    profiles/r02/serving_steps/table_timing_*)."""
    return cfg.get("table_timing", "step" if cfg["granularity"] == "layer" else "pass")


def step_down(rate: float, ratio: float) -> float:
    """Next offered rate after a timed run missed the 0.90 on-time bar: 4%
    lower near the bar, proportionally more far below it (a run far past
    saturation says little about where the bar is)."""
    if ratio >= 0.8:
        return rate * 0.96
    if ratio >= 0.5:
        return rate * 0.85
    return rate * 0.7


def capacity_search(serve, est: float, min_runs: int, max_runs: int = 14):
    """Largest offered rate with on-time >= 0.90 (the reference's capacity
    rule, simulator.hpp:804-820), by geometric bracketing then bisection.
    serve(rate, run_index) -> on-time ratio. Returns (rate, [(rate, ratio)])."""
    runs = []
    lo = hi = None
    rate = 0.5 * est
    while len(runs) < max_runs:
        ok = serve(rate, len(runs))
        runs.append((rate, ok))
        if ok >= 0.90:
            lo = rate
            if hi is None:
                rate *= 1.4
                continue
        else:
            hi = rate
            if lo is None:
                rate *= 0.6
                continue
        if (hi - lo) / hi < 0.06 and len(runs) >= min_runs:
            break
        rate = 0.5 * (lo + hi)
    return (lo if lo is not None else rate), runs


def layer_rooflines(desc: dict, prof: dict, pk: dict, batches=(1, 8, 32, 90), tc_peak: float | None = None,
                    w_bytes: float = 4.0) -> dict:
    """Per-layer achieved GB/s and roofline fraction from the measured h_k(b)
    table (CUDA events around each layer, tools: Executor.profile_table).
    Algorithmic work per layer: bytes = weights + bias once +
    b x (in + out + residual) activations, fp32 (weights w_bytes each: 2 for
    the bf16 path); FLOPs = 2 b MACs. Ideal time = max(bytes / HBM peak,
    FLOPs / tensor peak of the precision); frac = ideal / measured."""
    tc_peak = tc_peak or pk["tf32_tflops"]
    net = desc["nets"][0]
    comp = {c["id"]: c for c in prof["components"]}
    times = [dict(L["runtime_ms"]) for cid in prof["dnns"][0]["stages"] for L in comp[cid]["layers"]]
    T = net["tensors"]

    def elems(ref, out_side, op):
        if ref[0] < 0:
            return 0.0
        t = T[ref[0]]
        hw = op["Ho"] * op["Wo"] if out_side else t["H"] * t["W"]
        return float(hw * ref[2])

    out = {}
    for b in batches:
        rows, sum_ideal, sum_ms = [], 0.0, 0.0
        for k, L in enumerate(net["layers"]):
            if b not in times[k]:
                continue
            by = fl = 0.0
            for oi in L["ops"]:
                op = net["ops"][oi]
                w = op["weight_floats"] + op["out"][2] if op["kind"] == "conv" else \
                    (op["weight_floats"] + op["in"][2] if op["kind"] == "dwconv" else 0.0)
                act = elems(op["in"], False, op) + elems(op["res"], True, op)
                act += op["in"][2] if op["kind"] == "avgpool" else (op["out"][2] if op["kind"] == "softmax"
                                                                    else elems(op["out"], True, op))
                by += w_bytes * op["weight_floats"] + 4.0 * (w - op["weight_floats"] + b * act) \
                    if op["kind"] == "conv" else 4.0 * (w + b * act)
                fl += op["flops"] * b
            ms = times[k][b]
            ideal = max(by / (pk["hbm_gbs"] * 1e9), fl / (tc_peak * 1e12)) * 1e3
            sum_ideal += ideal
            sum_ms += ms
            rows.append([L["name"], round(ms * 1e3, 1), round(by / (ms * 1e-3) / 1e9, 1),
                         round(fl / (ms * 1e-3) / 1e12, 2), round(ideal / ms, 4)])
        out[str(b)] = {"layers": rows, "sum_us": round(sum_ms * 1e3, 1),
                       "frac_of_roofline": round(sum_ideal / sum_ms, 4) if sum_ms else None}
    out["columns"] = ["layer", "us", "GB/s", "TFLOP/s", "roofline frac"]
    return out


def cpu_forward(suite: str, batches=(1, 10, 90)) -> dict:
    """The builder's CPU fp32 forward (oracle/torch_forward.py: batched
    torch.nn.functional on every host thread; weights from libbs_nets.so, no
    GPU library) in img/s per batch. Not reference code: batchsim has no
    forward pass (a step is a table lookup, simulator.hpp:702-721)."""
    import numpy as np
    import torch

    from oracle.torch_forward import TorchNet
    from paper_2304_09961_b200.executor import describe_suite, make_image, suite_weights
    d = describe_suite(suite)
    tn = TorchNet(d, 0, suite_weights(suite, d), dtype=torch.float32)
    n = d["nets"][0]
    out = {"threads": torch.get_num_threads()}
    for b in batches:
        x = np.stack([make_image(1, i, n["in_H"], n["in_W"], n["in_C"]) for i in range(b)])
        tn.forward(x[:1])
        t = time.perf_counter()
        tn.forward(x)
        out[str(b)] = round(b / (time.perf_counter() - t), 2)
    return out


def reference_baseline(job: dict, rate: float, k: int, seed0: int) -> dict:
    """cpu_baseline of our line: the reference's run_sim on one host core for
    k runs of the timed workload (same table, trace seeds, deadline)."""
    rr = ref_runs(job, [{"rate": rate, "seed": seed0 + i} for i in range(k)])
    wall = sum(r["wall_ms"] for r in rr)
    plans = sum(r["schedules_computed"] for r in rr)
    gen = sum(r["generated"] for r in rr)
    return {"value": round(gen / (wall / 1000.0), 1), "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"{k} x {rr[0]['generated']} requests of the timed workload through the reference's run_sim "
                      f"(oracle/_ref/ref_dump, batchsim compiled unmodified, taskset -c 0) on this table; value = "
                      f"requests resolved per host second (a step is a table lookup there: no layer math)",
            "served_rps_simulated": round(sum(r["completed"] for r in rr) / (sum(r["span_ms"] for r in rr) / 1000.0), 1),
            "on_time_ratio_simulated": round(sum(r["on_time"] for r in rr) / max(1, gen), 4),
            "per_plan_ms": round(wall / max(1, plans), 4), "run_sim_wall_ms": round(wall / k, 2),
            "cpu": cpu_model(), "nproc": os.cpu_count()}


def run_reference(a, ws, rank) -> dict | None:
    """--impl reference: the reference's own CPU implementation of the path —
    batchsim's scheduler + event loop (run_sim, simulator.hpp:787-792;
    tardy_dp, deadline.hpp:130-282), compiled unmodified into
    oracle/_ref/ref_dump — on the same config: the latency table measured on
    a B200 by this repo (profiles/r02, the table our arm re-measures at
    startup), D = 6.25 x T1, the same arrival generator and seeds, the same
    capacity search and timed runs. batchsim executes no layers (a step is a
    cost-table lookup), so its served requests/s is the value of the metric
    in its simulated time; the host wall time of computing it is reported
    beside it (cores = 1: the reference is single-threaded). No library of
    this repo's executor is loaded here."""
    if rank != 0:
        return None
    cfg = CONFIGS[a.config]
    table = TABLES.get(a.config)
    if table is None or not table.exists():
        return {"impl": "reference", "unavailable": f"no measured B200 table committed for config {a.config}"}
    prof = json.loads(table.read_text())
    prof.pop("tile_tune", None)
    prof.pop("_meta", None)
    mb = cfg["max_batch"]
    comp = {c["id"]: c for c in prof["components"]}

    def dnn_ms(d, b):
        return sum(dict(L["runtime_ms"])[b] for cid in d["stages"] for L in comp[cid]["layers"])

    t1 = max(dnn_ms(d, 1) for d in prof["dnns"])
    tmax = max(dnn_ms(d, mb) for d in prof["dnns"])
    deadline = a.deadline_ms if a.deadline_ms else cfg["deadline_ms"]  # the same fixed D as our arm
    sim = sim_config(cfg, mb)
    names = [d["id"] for d in prof["dnns"]]
    w = {"process": cfg["process"], "count": a.requests, "relative_deadline": deadline}
    if len(names) > 1:
        w["dnn_mix"] = [[n, 1.0 / len(names)] for n in names]
    job = dict(collab_inputs(cfg), profile=prof, sim=sim, workload=w)
    search_runs = []

    def serve(rate, i):
        # the same probe as our arm: three traces per rate
        rs = ref_runs(job, [{"rate": rate, "seed": 1000 + 10 * i + s} for s in range(3)])
        search_runs.extend(rs)
        return sum(r["on_time"] for r in rs) / max(1, sum(r["generated"] for r in rs))

    cap_search, warm = capacity_search(serve, mb / tmax * 1000.0, a.warmup)
    cap = cap_search * 0.97
    retimed = []
    for attempt in range(7):  # the same timed-region rule as our arm
        timed = ref_runs(job, [{"rate": cap, "seed": 5000 + k} for k in range(a.steps)])
        ratio = sum(r["on_time"] for r in timed) / max(1, sum(r["generated"] for r in timed))
        if ratio >= 0.90 or attempt == 6:
            break
        retimed.append([round(cap, 1), round(ratio, 4)])
        cap = step_down(cap, ratio)
    completed = sum(r["completed"] for r in timed)
    span = sum(r["span_ms"] for r in timed)
    wall = sum(r["wall_ms"] for r in timed)
    plans = sum(r["schedules_computed"] for r in timed)
    gen = sum(r["generated"] for r in timed)
    value = completed / (span / 1000.0)
    sample = (f"{a.steps} timed runs x {a.requests} requests at 0.97 x the simulated capacity, after "
              f"{len(warm)} capacity-search runs; reference run_sim on 1 host core")
    return {"metric": METRIC if a.config == 2 else
            f"served requests/s ({cfg['process']}, on-time >= 0.90 capacity point), config {a.config}",
            "value": round(value, 2), "unit": UNIT, "impl": "reference", "n_gpus": ws,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(wall / a.steps, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64 (host scheduler; no layer math)", "data": "synthetic arrivals (reference generator)",
            "value_semantics": "served req/s of batchsim's run_sim in its simulated time on the measured B200 "
                               "table (what the reference reports for this metric); ms_per_step = host wall ms",
            "on_time_ratio": round(sum(r["on_time"] for r in timed) / max(1, gen), 4),
            "config": {"workload": cfg["workload"], "suite": cfg["suite"], "offered_rate_per_gpu": round(cap, 1),
                       "capacity_search_rate": round(cap_search, 1), "requests_per_step": a.requests,
                       "deadline_ms": round(deadline, 4), "t1_ms": round(t1, 4), "t_max_batch_ms": round(tmax, 4),
                       "max_batch": mb, "table": str(table.relative_to(ROOT)),
                       "parallelism": "reference is single-threaded (1 host core)"},
            "capacity_search": [[round(r, 1), round(x, 4)] for r, x in warm],
            "retimed_below_target": retimed,
            "host": {"run_sim_wall_ms_per_step": round(wall / a.steps, 2),
                     "per_plan_ms": round(wall / max(1, plans), 4),
                     "requests_per_host_second": round(gen / (wall / 1000.0), 1),
                     "cpu": cpu_model(), "nproc": os.cpu_count(), "cores_used": 1},
            "cpu_forward_img_s": cpu_forward(cfg["suite"]) if a.config == 2 else None,
            "cpu_baseline": {"value": round(value, 2), "unit": UNIT, "cores": 1, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": round(value, 2), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--requests", type=int, default=3000, help="requests per timed step")
    ap.add_argument("--warm-requests", type=int, default=3000, help="requests per capacity-search run")
    ap.add_argument("--slots", type=int, default=4096, help="activation-arena slots")
    ap.add_argument("--precision", default="tf32x2", choices=["tf32x2", "tf32", "bf16"])
    ap.add_argument("--stats-every", type=int, default=32,
                    help="sample every Nth launch with CUDA events in the timed region (every 4th cost ~13%% of config 2 capacity: an event between two kernels breaks their programmatic launch)")
    ap.add_argument("--cpu-forward", type=int, default=1, help="time the CPU fp32 forward at b = 1 / 10 / 90")
    ap.add_argument("--dump-table", default=None, help="write the measured latency table here")
    ap.add_argument("--table-flush-l2", type=int, default=0,
                    help="measure the scheduler's latency table with L2 flushed before every timed layer (cold)")
    ap.add_argument("--deadline-ms", type=float, default=None, help="override D = 6.25 x T1")
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS),
                    help="BASELINE.json config to serve (2 = the headline line)")
    a = ap.parse_args()
    a.warmup = max(3, a.warmup)
    ws, rank, local = dist_init()
    out = run_reference(a, ws, rank) if a.impl == "reference" else run_ours(a, ws, rank, local)
    if out is not None:
        print(json.dumps(out), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
