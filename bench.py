#!/usr/bin/env python
"""Benchmark: fused attention forward TFLOP/s on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  (N > 1: one rank per GPU over NCCL; launched by torch.distributed.run, or — when no
  WORLD_SIZE is set — bench.py starts the N ranks itself the same way. A world size that
  differs from --gpus is an error.)

A step = one tl_attn_fwd over this rank's shard of the workload (the whole hot path:
TMA loads, QK^T, online softmax, PV, epilogue — one kernel launch). Workload: C5
(B=64 Hq=Hkv=32 S=2048 D=128 bf16 causal — the BASELINE config sharded across
1/2/4/8 B200), head-sharded; the global problem is fixed, so scaling is "strong".
value = global FLOP (FA convention, x1/2 causal) / max-over-ranks device time.
Inputs (3.2 GB at N=1, >= 400 MB per rank at N=8) exceed the 126 MB L2, so no flush.

--impl reference times the fp64 CPU oracle (the tier's reference arm) on bounded
samples of the same workload, on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_17577_b200.configs import CONFIGS  # noqa: E402

METRIC = "attention fwd TFLOP/s (device-timed) and % of B200 bf16 tensor peak, 1/2/4/8 GPU"
UNIT = "TFLOP/s"
FALLBACK_PEAK_TFLOPS = 1590.0  # B200_PROFILING.md fallback (burst), used only if MEASURED_PEAKS.json is absent


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="C5", choices=sorted(CONFIGS))
    ap.add_argument("--shard", choices=["head", "batch"], default="head")
    ap.add_argument("--gather", action="store_true",
                    help="N>1: also time the replicated output: NCCL all-gather of O after the "
                         "kernel vs the fused replicated epilogue (tl_attn_fwd_replicated)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-extra", action="store_true", help="skip the other-config lines")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--clock-period-ms", type=float, default=5.0,
                    help="NVML clock sampling period during the timed region (0 = off)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo only to exercise N>1 on one GPU)")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return {"burst": float(p["bf16_tflops"]), "sustained": float(p["bf16_tflops_sustained"]),
                "hbm": float(p["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"burst": FALLBACK_PEAK_TFLOPS, "sustained": 1400.0, "hbm": 6650.0,
                "source": "fallback (B200_PROFILING.md)"}


# ------------------------------------------------------------------ clocks sampler
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, dev_index, period=0.005):
        self.samples, self.reasons, self.period = [], 0, period
        self.max_mhz = None
        self._stop = threading.Event()
        self.nv = None
        if period <= 0:
            return
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if self.nv is None or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        reasons = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------ helpers
def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """--gpus N > 1 without a torchrun environment: start the N ranks ourselves (one
    process per GPU, rendezvous on 127.0.0.1) under torch.distributed.run and return its
    exit code. The launched command is the driver's own form: `torchrun ... bench.py ...`."""
    import subprocess
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        # the job must have exactly --gpus ranks: a silent 1-rank run of `--gpus 8` would
        # report a 1-GPU number as an 8-GPU one
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started WORLD_SIZE={world} "
                         "ranks")
    if world > 1 and args.impl == "reference":
        return world, rank, local  # rank 0 runs the CPU oracle, the others exit; no process group
    if world > 1:
        import torch.distributed as dist
        if args.impl == "ours" and args.backend == "nccl" and torch.cuda.device_count() < world:
            raise SystemExit(f"bench.py: {world} NCCL ranks need {world} GPUs, "
                             f"{torch.cuda.device_count()} visible")
        if args.impl == "ours":
            # one rank per GPU; with fewer GPUs than ranks (gloo test mode) ranks share devices
            torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    elif args.impl == "ours":
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def time_device(fn, steps, warmup, world, per_launch_events=True):
    """W untimed steps, then K steps bracketed by barrier + synchronize; CUDA events on the
    launching (current) stream. Returns (total_ms max over ranks, mean per-launch kernel ms)."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)] if per_launch_events else []
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for i in range(steps):
        if per_launch_events:
            ev[i][0].record(stream)
        fn()
        if per_launch_events:
            ev[i][1].record(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    total = t0.elapsed_time(t1)
    kern = float(np.mean([a.elapsed_time(b) for a, b in ev])) if ev else total / steps
    return max_over_ranks(total, world), max_over_ranks(kern, world)


# ------------------------------------------------------------------ oracle (CPU) timing
def cpu_oracle_sample(cfg, seconds_min=8.0, seconds_max=25.0, heads_per_round=None):
    """Time the fp64 oracle (as it stands) on whole (b, h) heads of the workload, all host
    cores, until >= seconds_min of work. Returns dict with TFLOP/s."""
    import oracle
    from paper_2504_17577_b200.inputs import gen_qkv, to_bits

    cores = len(os.sched_getaffinity(0))
    heads_per_round = heads_per_round or cores
    q, k, v = gen_qkv(cfg.B, cfg.Hq, cfg.Hkv, cfg.Sq, cfg.Skv, cfg.D, cfg.dtype, cfg.seed, "cpu",
                      b_slice=slice(0, 1))
    qb, kb, vb = to_bits(q), to_bits(k), to_bits(v)
    odt = oracle.ORACLE_BF16 if cfg.dtype == torch.bfloat16 else oracle.ORACLE_F16
    one = cfg.__class__(**{**cfg.__dict__, "B": 1, "Hq": 1, "Hkv": 1})
    flop_head = one.flops()
    rows = list(range(cfg.Sq))
    done_flop, t0, rounds = 0.0, time.perf_counter(), 0
    while True:
        work = [(0, (rounds * heads_per_round + i) % cfg.Hq, rows) for i in range(heads_per_round)]
        oracle.attn_rows_parallel(qb, kb, vb, odt, int(cfg.causal), cfg.scale, work, threads=cores)
        done_flop += flop_head * len(work)
        rounds += 1
        el = time.perf_counter() - t0
        if el >= seconds_min or el >= seconds_max:
            break
    return {"value": done_flop / el / 1e12, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{rounds * heads_per_round} whole (b=0, h) heads of {cfg.name} "
                      f"({cfg.Sq}x{cfg.Skv}, D={cfg.D}, causal={cfg.causal}), all rows, fp64, "
                      f"{cores} threads, {el:.1f} s",
            "seconds": el}


def run_reference(args, world, rank):
    if rank != 0:
        return
    cfg = CONFIGS[args.workload]
    import oracle
    from paper_2504_17577_b200.inputs import gen_qkv, to_bits
    cores = len(os.sched_getaffinity(0))
    q, k, v = gen_qkv(cfg.B, cfg.Hq, cfg.Hkv, cfg.Sq, cfg.Skv, cfg.D, cfg.dtype, cfg.seed, "cpu",
                      b_slice=slice(0, 1))
    qb, kb, vb = to_bits(q), to_bits(k), to_bits(v)
    odt = oracle.ORACLE_BF16 if cfg.dtype == torch.bfloat16 else oracle.ORACLE_F16
    one = cfg.__class__(**{**cfg.__dict__, "B": 1, "Hq": 1, "Hkv": 1})
    # one step = one whole (b, h) head per core (bounded sample of the workload)
    nrows = cfg.Sq
    rows = list(range(nrows))

    def step(i):
        work = [(0, (i * cores + c) % cfg.Hq, rows) for c in range(cores)]
        oracle.attn_rows_parallel(qb, kb, vb, odt, int(cfg.causal), cfg.scale, work, threads=cores)
        return one.flops() * cores

    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    flop = sum(step(args.warmup + i) for i in range(args.steps))
    el = time.perf_counter() - t0
    val = flop / el / 1e12
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": el / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {**cfg.as_dict(), "sample": "per step: one whole (b=0,h) head per core"},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{args.steps} steps x {cores} whole heads of {cfg.name}"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0, "world_size": world}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def run_ours(args, world, rank, local):
    from paper_2504_17577_b200 import (HostAttention, attention, load_library,
                                       tl_attn_last_launch_count)
    from paper_2504_17577_b200 import build as pkg_build
    from paper_2504_17577_b200.dist import gather_output, make_shard
    from paper_2504_17577_b200.inputs import gen_qkv

    if rank == 0 and pkg_build.needs_build():
        pkg_build.build()
    barrier(world)
    load_library()
    cfg = CONFIGS[args.workload]
    pk = peaks()
    shard = make_shard(args.shard, rank, world, cfg.B, cfg.Hq, cfg.Hkv)
    q, k, v = gen_qkv(cfg.B, cfg.Hq, cfg.Hkv, cfg.Sq, cfg.Skv, cfg.D, cfg.dtype, cfg.seed, "cuda",
                      b_slice=shard.b, hq_slice=shard.hq, hkv_slice=shard.hkv)
    Bl, Sq, Hql, D = q.shape
    Hkvl = k.shape[2]
    o = torch.empty_like(q)
    lse = torch.empty((Bl, Hql, Sq), dtype=torch.float32, device="cuda")
    launches = [0]

    def step():
        attention(q, k, v, causal=cfg.causal, scale=cfg.scale, out=o, lse_out=lse)
        launches[0] += tl_attn_last_launch_count()  # kernels this call launched (1)

    with ClockSampler(local, args.clock_period_ms / 1000.0) as clk:
        total_ms, kern_ms = time_device(step, args.steps, args.warmup, world)
    timed_launches = launches[0] - args.warmup * tl_attn_last_launch_count()
    flop = cfg.flops()
    ms = total_ms / args.steps
    value = flop / (ms * 1e-3) / 1e12
    # dominant kernel (the only one): per-launch algorithmic FLOP / mean launch duration
    flop_local = flop / world
    achieved = flop_local / (kern_ms * 1e-3) / 1e12
    roofline = {"bound": "tensor", "achieved": achieved, "peak": pk["burst"], "unit": UNIT,
                "frac": achieved / pk["burst"], "traffic": ncu_traffic(cfg.name, world),
                "peak_source": pk["source"] + " bf16 burst",
                "kernel": ("tl_attn_fwd_kernel_2sm<bf16> (CTA pair)" if cfg.D == 128
                           else f"tl_attn_fwd_kernel<{cfg.D},{cfg.dtype_name}>"),
                "frac_of_sustained": achieved / pk["sustained"],
                "frac_of_spec_2250": achieved / 2250.0}
    # the softmax's own floor: every allowed (query, key) pair needs one exp2,
    # 16 per clock per SM on MUFU, at the median SM clock measured during the timed region
    ck = clk.summary()
    mhz = ck.get("sm_mhz") or ck.get("sm_max_mhz")
    if mhz:
        n_sm = torch.cuda.get_device_properties(local).multi_processor_count
        floor_ms = cfg.flops_exact() / world / (4.0 * cfg.D) / (n_sm * 16 * mhz * 1e6) * 1e3
        roofline["mufu_floor_ms"] = floor_ms
        roofline["frac_of_mufu_floor"] = floor_ms / kern_ms

    gather_ms = None
    if args.gather and world > 1:
        import torch.distributed as dist
        for _ in range(2):
            gather_output(o, lse, shard)
        torch.cuda.synchronize()
        dist.barrier()
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            gather_output(o, lse, shard)
        b_.record()
        torch.cuda.synchronize()
        gather_ms = max_over_ranks(a.elapsed_time(b_) / 3, world)
        # fused alternative: the kernel's epilogue stores every O tile into all
        # ranks' full buffers (P2P over NVLink) + device flag barriers; time per call
        # (attention + replication) next to attention + NCCL all-gather
        from paper_2504_17577_b200.dist import ReplicatedOutput
        rep = ReplicatedOutput(shard, cfg.B, cfg.Sq, cfg.Hq, cfg.D, cfg.dtype)

        def fused():
            rep(q, k, v, causal=cfg.causal, scale=cfg.scale)

        def unfused():
            step()
            gather_output(o, lse, shard)

        f_total, _ = time_device(fused, 5, 2, world, per_launch_events=False)
        u_total, _ = time_device(unfused, 5, 2, world, per_launch_events=False)
        gather_ms = {"nccl_all_gather_ms": gather_ms, "attn_plus_nccl_gather_ms": u_total / 5,
                     "attn_fused_replicated_ms": f_total / 5}
        rep.close()

    # ---- end to end through the public host-buffer entry (H2D + kernel + D2H per step)
    e2e = None
    if args.e2e_steps > 0:
        qh, kh, vh = (t.cpu().pin_memory() for t in (q, k, v))
        oh = torch.empty(qh.shape, dtype=qh.dtype).pin_memory()
        lh = torch.empty((Bl, Hql, Sq), dtype=torch.float32).pin_memory()
        ha = HostAttention(Bl, Hql, Hkvl, Sq, cfg.Skv, D, with_lse=True)

        def estep():
            ha(qh, kh, vh, oh, lh, causal=cfg.causal, scale=cfg.scale)

        e_total, _ = time_device(estep, args.e2e_steps, 1, world, per_launch_events=False)
        e_ms = e_total / args.e2e_steps
        h2d = sum(t.numel() * t.element_size() for t in (qh, kh, vh))
        d2h = oh.numel() * oh.element_size() + lh.numel() * 4
        # transfer floor of the same bytes: pinned-memory copies alone (one H2D of q's size
        # and one D2H of o's size, timed like the step), scaled to the step's byte counts
        floor = pcie_floor(qh, oh, h2d, d2h)
        e2e = {"value": flop / (e_ms * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
               "steps": args.e2e_steps, "api": "tl_attn_fwd_host (pinned host buffers)",
               **floor, "frac_of_transfer_floor": floor["transfer_floor_ms"] / e_ms}
        del qh, kh, vh, oh, lh, ha

    extra = {}
    if not args.no_extra and world == 1:
        del q, k, v, o, lse
        torch.cuda.empty_cache()
        for name in ("C1", "C2", "C3", "C4", "T0"):
            if name == cfg.name:
                continue
            extra[name] = bench_one(CONFIGS[name], pk, steps=max(5, min(args.steps, 20)))
        from paper_2504_17577_b200.configs import PAPER_T3
        for name in ("FA0", "FA1", "FA2", "FA3", "FA4"):  # the paper's FlashAttention shapes (Table 3)
            extra["paper_" + name] = bench_one(PAPER_T3[name], pk, steps=max(5, min(args.steps, 20)),
                                               graph=True)
        for gname in ("M5", "M2", "V1", "V4"):  # the paper's GEMM on Table 2 shapes
            extra["gemm_" + gname] = bench_gemm(gname, pk)
        from paper_2504_17577_b200.configs import MLA_CONFIGS
        for mc in MLA_CONFIGS:  # MLA decode (Fig. 18)
            extra["mla_" + mc.name] = bench_mla(mc, pk, steps=max(5, min(args.steps, 20)))
        from paper_2504_17577_b200.configs import SSD_CONFIGS
        for sname in ("CT5", "CC5", "CT3", "CC3"):  # Mamba-2 SSD (Table 4)
            extra["ssd_" + sname] = bench_ssd(SSD_CONFIGS[sname], pk, steps=max(5, min(args.steps, 10)))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_oracle_sample(cfg)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": cfg.dtype_name, "data": "synthetic",
                "config": {**cfg.as_dict(), "parallelism": f"{args.shard}-shard x{world}",
                           "flop_per_step": flop, "flop_convention": "4*B*Hq*Sq*Skv*D, x1/2 causal",
                           "exact_flop_per_step": cfg.flops_exact(),
                           "exact_tflops": cfg.flops_exact() / (ms * 1e-3) / 1e12,
                           "l2": "inputs > 126 MB L2 (no flush)"},
                "frac_of_peak": value / pk["burst"],
                "roofline": roofline,
                "clocks": clk.summary(),
                "e2e": e2e,
                "gpu_launches": timed_launches,
                "cpu_baseline": cpu,
                "gather_ms": gather_ms,
                "also": extra}
        print(json.dumps(line), flush=True)


def pcie_floor(src_h, dst_h, h2d_bytes, d2h_bytes):
    """Measured pinned host<->device copy bandwidth (one copy each way, CUDA events) and the
    resulting floor for a step that moves h2d_bytes up and d2h_bytes down with the two
    directions overlapped (the host entry pipelines them): max(h2d/bw_up, d2h/bw_down)."""
    dev = torch.empty(src_h.shape, dtype=src_h.dtype, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    dev.copy_(src_h, non_blocking=True)
    torch.cuda.synchronize()
    ev[0].record()
    dev.copy_(src_h, non_blocking=True)
    ev[1].record()
    ev[2].record()
    dst_h.copy_(dev, non_blocking=True)
    ev[3].record()
    torch.cuda.synchronize()
    up = src_h.numel() * src_h.element_size() / (ev[0].elapsed_time(ev[1]) * 1e-3) / 1e9
    down = dst_h.numel() * dst_h.element_size() / (ev[2].elapsed_time(ev[3]) * 1e-3) / 1e9
    del dev
    return {"h2d_gbs_measured": up, "d2h_gbs_measured": down,
            "transfer_floor_ms": max(h2d_bytes / up, d2h_bytes / down) / 1e6}


def ncu_traffic(name, world):
    """DRAM bytes per launch from the committed ncu --set full summary, if one exists."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(name, {}).get(str(world))
    except Exception:
        return None


# The `also` block times every config from the same starting state: 0.3 s of idle GPU after
# its inputs are generated (input generation and the previous config heat the chip into its
# power limit, which otherwise lands on whichever config comes next).
ALSO_IDLE_S = 0.3


def settle():
    torch.cuda.synchronize()
    time.sleep(ALSO_IDLE_S)


def bench_one(cfg, pk, steps=20, warmup=3, graph=False):
    from paper_2504_17577_b200 import attention
    from paper_2504_17577_b200.inputs import gen_qkv
    q, k, v = gen_qkv(cfg.B, cfg.Hq, cfg.Hkv, cfg.Sq, cfg.Skv, cfg.D, cfg.dtype, cfg.seed, "cuda")
    o = torch.empty_like(q)
    lse = torch.empty((cfg.B, cfg.Hq, cfg.Sq), dtype=torch.float32, device="cuda")
    small = cfg.hbm_bytes() < 64e6
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if small else None

    def call():
        attention(q, k, v, causal=cfg.causal, scale=cfg.scale, out=o, lse_out=lse)

    settle()
    for _ in range(warmup):
        call()
    st = torch.cuda.current_stream()
    evs = []
    with ClockSampler(torch.cuda.current_device(), period=0.002) as clk:
        for _ in range(steps):
            if flush is not None:
                flush.zero_()  # write > L2 between launches for L2-resident shapes
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            call()
            b.record(st)
            evs.append((a, b))
        torch.cuda.synchronize()
    kern_ms = float(np.median([a.elapsed_time(b) for a, b in evs]))
    tf = cfg.flops() / (kern_ms * 1e-3) / 1e12
    res = {"tflops": tf, "kernel_ms": kern_ms, "frac_of_peak": tf / pk["burst"],
           "hbm_gbs": cfg.hbm_bytes() / (kern_ms * 1e-3) / 1e9, **cfg.as_dict()}
    # MUFU-only softmax floor: one exp2 per allowed (query, key) pair at 16 ex2 / clock / SM
    # (the SFU rate, B200_PROFILING / r02 notes) and the median SM clock of this run
    ck = clk.summary()
    mhz = ck.get("sm_mhz") or ck.get("sm_max_mhz")
    if mhz:
        n_exp = cfg.flops_exact() / (4.0 * cfg.D)
        n_sm = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        floor_ms = n_exp / (n_sm * 16 * mhz * 1e6) * 1e3
        res.update({"mufu_floor_ms": floor_ms, "frac_of_mufu_floor": floor_ms / kern_ms,
                    "mufu_floor_clock_mhz": mhz})
    res["clocks"] = {k: ck.get(k) for k in ("sm_mhz", "reasons")}
    res["idle_before_s"] = ALSO_IDLE_S
    if small:
        res["note"] = "L2 flushed between launches (256 MB write)"
    if graph:
        # device time per launch without host launch cost: 20 back-to-back calls in one CUDA
        # graph (inputs L2-warm), replayed 5 times
        s_ = torch.cuda.Stream()
        s_.wait_stream(st)
        with torch.cuda.stream(s_):
            call()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s_):
            for _ in range(20):
                call()
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(5):
            g.replay()
        b.record(st)
        torch.cuda.synchronize()
        gms = a.elapsed_time(b) / 100
        res["graph_us"] = gms * 1e3
        res["graph_tflops"] = cfg.flops() / (gms * 1e-3) / 1e12
        res["graph_note"] = "CUDA graph of 20 back-to-back launches, L2-warm, device time per launch"
        del g
    del q, k, v, o, lse
    torch.cuda.empty_cache()
    return res


def bench_mla(cfg, pk, steps=20, warmup=3):
    """tl_mla_decode on an MLA config (inputs > L2). Bound: HBM (the latent cache is read
    once; 235 FLOP/B at 128 heads is just below the bf16 ridge, 30 FLOP/B at 16 heads)."""
    from paper_2504_17577_b200 import (mla_decode, tl_attn_last_launch_count,
                                       tl_mla_decode_workspace_bytes)
    from paper_2504_17577_b200.inputs import gen_mla
    q, qp, kv, kp = gen_mla(cfg.B, cfg.H, cfg.Hkv, cfg.Skv, cfg.Dl, cfg.Dr, cfg.dtype, cfg.seed,
                            "cuda")
    sl = cfg.seqlens()
    sld = None if sl is None else torch.as_tensor(sl, device="cuda")
    ws = torch.empty(tl_mla_decode_workspace_bytes(cfg.B, cfg.H, cfg.Hkv), dtype=torch.uint8,
                     device="cuda")
    o = torch.empty((cfg.B, cfg.H, cfg.Dl), dtype=cfg.dtype, device="cuda")
    lse = torch.empty((cfg.B, cfg.H), dtype=torch.float32, device="cuda")

    def call():
        mla_decode(q, qp, kv, kp, seqlens=sld, out=o, lse_out=lse, workspace=ws)

    settle()
    for _ in range(warmup):
        call()
    st = torch.cuda.current_stream()
    evs = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        call()
        b.record(st)
        evs.append((a, b))
    torch.cuda.synchronize()
    ms = float(np.median([a.elapsed_time(b) for a, b in evs]))
    gbs = cfg.hbm_bytes() / (ms * 1e-3) / 1e9
    tf = cfg.flops() / (ms * 1e-3) / 1e12
    res = {"us": ms * 1e3, "hbm_gbs": gbs, "frac_of_hbm": gbs / pk["hbm"], "tflops": tf,
           "frac_of_peak": tf / pk["burst"], "launches_per_call": tl_attn_last_launch_count(),
           "bound": "hbm", **cfg.as_dict()}
    del q, qp, kv, kp, o, lse, ws
    torch.cuda.empty_cache()
    return res


def bench_ssd(cfg, pk, steps=10, warmup=3):
    """Mamba-2 SSD chunk_state (CT) / chunk_scan (CC) on a Table 4 shape (PAPER.md
    P:L464-478). Bound: HBM (80-97 FLOP/B); GB/s of the algorithmic bytes (every input read
    once, the output written once; configs.SsdConfig.hbm_bytes)."""
    from paper_2504_17577_b200 import ssd_chunk_scan, ssd_chunk_state, tl_attn_last_launch_count
    from paper_2504_17577_b200.inputs import gen_ssd, gen_ssd_cb_prev, ssd_chunked_dt
    x, Bm, C, dtv, A, D = gen_ssd(cfg.B, cfg.L, cfg.H, cfg.G, cfg.P, cfg.N, cfg.dtype, cfg.seed,
                                  "cuda")
    dt, dA = ssd_chunked_dt(dtv, A, cfg.Q)
    if cfg.kind == "state":
        out = torch.empty((cfg.B, cfg.nc, cfg.H, cfg.P, cfg.N), dtype=cfg.dtype, device="cuda")

        def call():
            ssd_chunk_state(x, Bm, dt, dA, out=out)
    else:
        cb, prev = gen_ssd_cb_prev(cfg.B, cfg.L, cfg.H, cfg.G, cfg.P, cfg.N, cfg.dtype, cfg.seed,
                                   "cuda")
        out = torch.empty_like(x)

        def call():
            ssd_chunk_scan(cb, x, dt, dA, C, prev, D, out=out)
    settle()
    for _ in range(warmup):
        call()
    st = torch.cuda.current_stream()
    evs = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        call()
        b.record(st)
        evs.append((a, b))
    torch.cuda.synchronize()
    ms = float(np.median([a.elapsed_time(b) for a, b in evs]))
    gbs = cfg.hbm_bytes() / (ms * 1e-3) / 1e9
    res = {"us": ms * 1e3, "hbm_gbs": gbs, "frac_of_hbm": gbs / pk["hbm"],
           "tflops": cfg.flops() / (ms * 1e-3) / 1e12, "bound": "hbm",
           "launches_per_call": tl_attn_last_launch_count(), **cfg.as_dict()}
    del x, Bm, C, out
    torch.cuda.empty_cache()
    return res


GEMM_TABLE2 = {"M2": (4096, 28672, 8192), "M5": (8192, 8192, 8192),  # PAPER.md Table 2
               "V1": (1, 43008, 14336), "V4": (1, 14336, 57344)}     # GEMV rows (HBM-bound)


def bench_gemm(name, pk, iters=10):
    """tl_gemm (bf16) on a Table 2 shape, with cuBLAS (torch.matmul) timed as context."""
    from paper_2504_17577_b200 import gemm
    from paper_2504_17577_b200.inputs import gen_tensor
    M, N, K = GEMM_TABLE2[name]
    a = gen_tensor((M, K), 2024, "q", torch.bfloat16, "cuda")
    b = gen_tensor((K, N), 2024, "k", torch.bfloat16, "cuda")
    c = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")

    def med(fn):
        settle()
        for _ in range(3):
            fn()
        evs = []
        for _ in range(iters):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            evs.append((e0, e1))
        torch.cuda.synchronize()
        return float(np.median([x.elapsed_time(y) for x, y in evs]))

    t = med(lambda: gemm(a, b, out=c))
    tc = med(lambda: torch.matmul(a, b, out=c))
    fl = 2.0 * M * N * K
    del a, b, c
    torch.cuda.empty_cache()
    res = {"shape": [M, N, K], "tflops": fl / t / 1e9, "kernel_ms": t,
           "frac_of_peak": fl / t / 1e9 / pk["burst"], "cublas_tflops": fl / tc / 1e9,
           "vs_cublas": tc / t}
    if M == 1:  # GEMV: HBM-bound, the roofline is the copy bandwidth
        by = 2.0 * (K + K * N + N)
        res.update({"bound": "hbm", "hbm_gbs": by / t / 1e6, "frac_of_hbm": by / t / 1e6 / pk["hbm"],
                    "cublas_hbm_gbs": by / tc / 1e6})
    return res


def main():
    args = parse()
    if args.gpus < 1:
        raise SystemExit("bench.py: --gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    world, rank, local = dist_setup(args)
    try:
        if args.impl == "reference":
            run_reference(args, world, rank)
        else:
            run_ours(args, world, rank, local)
    finally:
        import torch.distributed as dist
        if world > 1 and dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
