#!/usr/bin/env python3
"""Benchmark: exactly summed doubles/s on B200 (BASELINE.json metric), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4|c2|c5|...] [--impl ours|reference]

Default workload: BASELINE.json config c4, the one its metric ("at 1/2/4/8 B200") is quoted
on: n = 2^33 doubles (64 GiB), seed 4, exponent U[-1022,1023], split into N contiguous shards,
one per GPU (strong scaling). A step is one pass of the whole hot path (SURVEY.md §8(a) rows
a1-a8) over the whole input:
  N = 1: one fused launch of xsum_sum (decompose + lane-column accumulate + regularize +
         block/grid merge + canonicalize + round) over the 64 GiB in HBM.
  N > 1: (torchrun, one process per GPU) every rank sums its shard and the 384-byte states are
         exchanged and merged: ONE launch per rank with the exchange over
         NVLink peer memory (xsum_sum_allreduce), or, if that is unavailable or fails its checks
         (probe before timing; every timed step's flags after it), the shard sums + an NCCL
         all-gather + xsum_merge_round.
Inputs are synthetic (synth/, the recipe in DESIGN.md) and larger than the 126 MB L2 (c1 flushes
it between steps). `--impl reference` times the CPU oracle instead (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "doubles/s exact-summed (device-timed) at 1/2/4/8 B200; % of HBM-read roofline"
UNIT = "doubles/s"
FMT_OF = {"c2f32": "binary32", "c2f16": "binary16", "c2bf16": "bfloat16"}


def metric_unit(cfg_name: str):
    """BASELINE.json's metric, or for the other-format workloads the same metric in their values."""
    if cfg_name in FMT_OF:
        return (f"{FMT_OF[cfg_name]} values/s exact-summed (device-timed); % of HBM-read roofline",
                f"{FMT_OF[cfg_name]} values/s")
    return METRIC, UNIT


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    # c1..c5: BASELINE.json configs; c5csr / c2f32 / c2f16 / c2bf16: measurement workloads of the
    # NEXT rows (CSR segments, other input formats; synth/gen.py)
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5", "c5csr", "c2f32", "c2f16",
                                                         "c2bf16", "c2dim0", "c5s16", "c2cs", "c3cs"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sustained-s", type=float, default=2.0,
                    help="after the timed region, run the step back to back this long and report the "
                         "power-capped rate as `sustained` (0: skip)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    # testing the N>1 host path with several ranks on ONE GPU (gloo, no fused exchange: no kernel
    # waits on another rank then); the driver's runs use the defaults
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--no-fused", action="store_true")
    return ap.parse_args()


def workload(cfg_name: str, world: int) -> dict:
    import synth
    cfg = synth.CONFIGS[cfg_name]
    desc = {
        "c1": "c1: n=2^20 doubles, seed 1, exponent U[-10,10]",
        "c2": "c2: n=2^28 doubles, seed 2, random sign, uniform mantissa, exponent U[-1000,1000]",
        "c3": "c3: 2^27 (a,-a) pairs exp U[0,600] + 2^20 tiny exp U[-900,-800], permuted, seed 3",
        "c4": "c4: n=2^33 doubles, seed 4, exponent U[-1022,1023], sharded over the GPUs",
        "c5": "c5: 2^16 segments x 2^12 doubles, seed 5, exponent U[-200,200]",
        "c5csr": "c5csr: 2^16 CSR segments of 1..8192 doubles (mean 4096), seed 9, exponent U[-200,200]",
        "c2f32": "c2f32: n=2^28 binary32, seed 6, uniform over the finite bit patterns",
        "c2f16": "c2f16: n=2^28 binary16, seed 7, uniform over the finite bit patterns",
        "c2bf16": "c2bf16: n=2^28 bfloat16, seed 8, uniform over the finite bit patterns",
        "c2dim0": "c2dim0: c2's 2^28 doubles as a [4096, 65536] matrix, exact_sum_dim over dim 0 (65536 sums)",
        "c5s16": "c5s16: 2^24 segments x 16 doubles, seed 10, exponent U[-200,200]",
        "c2cs": "c2cs: c2's 2^28 doubles, condition-number-sensitive sum (xsum_sum_condsens, rule 1)",
        "c3cs": "c3cs: c3's 2^28 + 2^20 doubles (ill-conditioned), condition-number-sensitive sum (rule 1)",
    }[cfg_name]
    if cfg_name == "c4":
        n_total = cfg["n"]
        scaling = "strong"
    else:
        n_total = cfg["n"] * world
        scaling = "weak"
    return dict(desc=desc, n_total=n_total, scaling=scaling, cfg=cfg)


# ------------------------------------------------------------------------------------------
# clocks during the timed region (NVML, fine-grained; the recipe's nvidia-smi fields)
# ------------------------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle",
               0x2: "applications_clocks_setting"}

    def __init__(self, index: int, period_s: float = 0.002):
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self.ok = False
        self._stop = threading.Event()
        self.period = period_s
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()
            try:  # one last sample right at the end of the region
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            except Exception:
                pass

    def summary(self) -> dict:
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and v != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


def clocks_rejected(c: dict) -> bool:
    """The timing rules' rejection test for one timed region's clock summary."""
    if not c.get("samples"):
        return False
    if set(c.get("reasons", [])) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}:
        return True
    mx, md = c.get("sm_max_mhz"), c.get("sm_mhz")
    return bool(mx and md and md < 0.75 * mx and not c.get("reasons"))


def measured_peak_hbm() -> tuple[float, str]:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, read+write)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def profiled_traffic(cfg_name: str):
    """dram read+write bytes per launch of the dominant kernel from the committed ncu --set full
    summary (profiles/ncu_summary.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as fh:
            s = json.load(fh)
        return s.get("traffic_bytes_per_launch", {}).get(cfg_name)
    except Exception:
        return None


# ------------------------------------------------------------------------------------------
# CPU oracle arm (cpu_baseline and --impl reference)
# ------------------------------------------------------------------------------------------
SEG_CFGS = ("c5", "c5csr", "c5s16", "c2dim0")


def oracle_segments_input(cfg_name: str):
    """The host input of a segmented workload in segment order: (x, offsets or None, seg_len)."""
    import numpy as np

    import synth
    cfg = synth.CONFIGS[cfg_name]
    if cfg_name == "c2dim0":                     # fibre i of the [4096, 65536] matrix = column i
        rows, cols = cfg["shape"]
        x = np.ascontiguousarray(synth.host_generate("c2").reshape(rows, cols).T)
        return x.reshape(-1), None, rows
    x = synth.host_generate(cfg_name)
    if cfg["kind"] == "csr":
        return x, synth.gen.csr_offsets(cfg).astype(np.uint64), None
    return x, None, cfg["seg_len"]


def oracle_rate(cfg_name: str, target_s: float = 1.5, max_n: int = 1 << 28):
    import numpy as np
    """Time the oracle (as it stands) on a bounded prefix of the workload on all host cores:
    passes over the same sample until ~target_s seconds of wall time (x the host cores =
    10-30 s of CPU work). Returns (doubles/s, cores, sample size, passes, seconds, config)."""
    import oracle
    import synth
    cores = oracle.host_threads()
    if cfg_name in SEG_CFGS:
        # the workload's own computation: every segment (fibre) summed and rounded on its own
        # (oracle.sum_segments), the whole input (input preparation untimed)
        x, off, L = oracle_segments_input(cfg_name)
        oracle.sum_segments(x[:L or 64], seg_len=L or 64, nthreads=cores)
        passes, t0 = 0, time.perf_counter()
        while True:
            ref = oracle.sum_segments(x, off, seg_len=L, nthreads=cores)
            passes += 1
            dt = time.perf_counter() - t0
            if dt >= target_s:
                break
        m = x.size
        del x
        return m * passes / dt, cores, m, passes, dt, cfg_name, ref
    gen_name = "c2" if cfg_name in ("c1",) else cfg_name
    m = min(max_n, synth.CONFIGS[gen_name]["n"])
    if synth.CONFIGS[gen_name]["kind"] == "cancel":
        # c3's device input is permuted: only the whole input has the same exact sum on the host
        m = synth.CONFIGS[gen_name]["n"]
    fmt = synth.CONFIGS[gen_name].get("fmt")
    if fmt is None:
        x = synth.host_generate(gen_name, 0, m)

        def run(a):
            return oracle.exact_sum(a, nthreads=cores)
    else:
        x = synth.host_bits(gen_name, 0, m)

        def run(a):
            if fmt == "f32":
                return oracle.exact_sum(a.view(np.float32), nthreads=cores)
            return oracle.exact_sum(a, nthreads=cores, fmt=fmt)
    run(x[: 1 << 16])                                       # load the library, warm the threads
    passes, t0 = 0, time.perf_counter()
    while True:
        ref = run(x)
        passes += 1
        dt = time.perf_counter() - t0
        if dt >= target_s:
            break
    del x
    return m * passes / dt, cores, m, passes, dt, gen_name, ref


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    import numpy as np

    import oracle
    import synth
    wl = workload(args.config, world)
    cores = oracle.host_threads()
    if args.config in SEG_CFGS:
        return run_reference_segments(args, wl, cores)
    rate, _, _, _, _, gen_name, _ = oracle_rate(args.config, target_s=0.5, max_n=1 << 24)
    budget = 90.0
    m = int(max(1 << 14, min(1 << 26, rate * budget / max(1, args.steps + args.warmup))))
    fmt = synth.CONFIGS[gen_name].get("fmt")
    if fmt is None:
        x = synth.host_generate(gen_name, 0, m)
    elif fmt == "f32":
        x = synth.host_bits(gen_name, 0, m).view(np.float32)
    else:
        x = synth.host_bits(gen_name, 0, m)
    kw = {"fmt": fmt} if fmt in ("f16", "bf16") else {}
    for _ in range(args.warmup):
        oracle.exact_sum(x, nthreads=cores, **kw)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.exact_sum(x, nthreads=cores, **kw)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = m * args.steps / tot
    sample = f"{gen_name} elements [0, {m}) per step (bounded sample of the workload), {cpu_model()}"
    metric, unit = metric_unit(args.config)
    line = {
        "impl": "reference", "metric": metric, "value": value, "unit": unit, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": wl["scaling"], "vs_baseline": None, "dtype": "int64",
        "data": "synthetic", "config": {"workload": wl["desc"], "sample_n": m},
        "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_reference_segments(args, wl, cores):
    """--impl reference for a segmented workload: each step sums and rounds a bounded prefix of
    whole segments with the oracle (oracle.sum_segments)."""
    import numpy as np

    import oracle
    x, off, L = oracle_segments_input(args.config)
    nseg_all = (off.size - 1) if off is not None else x.size // L
    budget_elems = int(max(1 << 16, min(x.size, 1.2e9 * 90 / max(1, args.steps + args.warmup))))
    if off is not None:
        k = int(np.searchsorted(off, budget_elems, side="right")) - 1
        k = max(1, min(nseg_all, k))
        xs, offs, m = x[: int(off[k])], off[: k + 1], int(off[k])
    else:
        k = max(1, min(nseg_all, budget_elems // L))
        xs, offs, m = x[: k * L], None, k * L
    for _ in range(args.warmup):
        oracle.sum_segments(xs, offs, seg_len=L, nthreads=cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.sum_segments(xs, offs, seg_len=L, nthreads=cores)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = m * args.steps / tot
    metric, unit = metric_unit(args.config)
    sample = f"{args.config}: the first {k} segments ({m} elements) per step, each summed and rounded, {cpu_model()}"
    line = {
        "impl": "reference", "metric": metric, "value": value, "unit": unit, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": wl["scaling"], "vs_baseline": None, "dtype": "int64",
        "data": "synthetic", "config": {"workload": wl["desc"], "sample_n": m, "sample_segments": k},
        "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------
def steps_verdict(xsum, rows, world: int, device) -> str | None:
    """Check every timed step's result record (rows: K x RESULT_BYTES uint8, host): the same bits
    and flags in every step and on every rank, and no XSUM_F_PEER_TIMEOUT in ANY step (a timed-out
    fused step spins ~2 s and returns a value that is not the group's sum). The decision is
    all-reduced so every rank agrees. Returns None if the steps are valid, else the reason."""
    import numpy as np
    import torch

    rs = [xsum.Result.from_bytes(np.asarray(r, dtype=np.uint8).tobytes()) for r in rows]
    flags_or = 0
    for r in rs:
        flags_or |= r.flags
    bits = {r.bits for r in rs}
    local_bad = 0
    if flags_or & xsum.F_PEER_TIMEOUT:
        local_bad |= 1
    if len(bits) != 1 or len({r.flags for r in rs}) != 1:
        local_bad |= 2
    b0 = rs[0].bits
    t = torch.tensor([b0 - (1 << 64) if b0 >> 63 else b0, rs[0].flags, local_bad], dtype=torch.int64, device=device)
    if world > 1:
        lo, hi = t.clone(), t.clone()
        allreduce_(lo, torch.distributed.ReduceOp.MIN)
        allreduce_(hi, torch.distributed.ReduceOp.MAX)
    else:
        lo = hi = t
    bad = int(hi[2])
    if bad & 1:
        steps = [i for i, r in enumerate(rs) if r.flags & xsum.F_PEER_TIMEOUT]
        return f"peer timeout in timed step(s) {steps[:8]} on this rank" if steps else \
            "peer timeout in a timed step on another rank"
    if bad & 2:
        return "results differ between timed steps"
    if int(lo[0]) != int(hi[0]) or int(lo[1]) != int(hi[1]):
        return "ranks disagree on the result"
    return None


def step_stats(ms: list[float]) -> dict:
    return {"median_ms": statistics.median(ms), "min_ms": min(ms), "max_ms": max(ms)}


def run_ours(args, rank: int, world: int, local_rank: int):
    import numpy as np
    import torch

    import paper_1605_05436_b200 as xsum
    import synth
    from paper_1605_05436_b200 import dist

    dev_index = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        import torch.distributed as tdist
        if args.dist_backend == "nccl":
            tdist.init_process_group("nccl", device_id=dev)
        else:
            tdist.init_process_group("gloo")
    xsum.build()
    synth.build()
    wl = workload(args.config, world)
    cfg = wl["cfg"]
    if world > 1 and (cfg["kind"] in ("bits", "csr") or args.config in ("c2dim0", "c5s16", "c2cs", "c3cs")):
        raise SystemExit(f"--config {args.config} is a one-GPU measurement workload")
    seg = args.config in ("c5", "c5csr", "c5s16", "c2dim0")      # many results per step
    csr = None
    metric, unit = metric_unit(args.config)

    # this rank's input, generated in HBM (untimed)
    if cfg["kind"] == "bits":
        x = synth.device_bits(args.config, device=dev)
    elif args.config == "c5csr":
        x = synth.device_generate("c5csr", device=dev)
        csr = synth.csr_offsets("c5csr", device=dev)
    elif args.config == "c4":
        start, stop = dist.shard_range(cfg["n"], rank, world)   # strong scaling: contiguous shards
        x = synth.device_generate("c4", start, stop - start, device=dev)
    elif args.config in ("c3", "c3cs"):
        x = synth.device_generate(args.config, device=dev)
    else:
        x = synth.device_generate(args.config, device=dev)   # same c-config per rank (weak scaling)
    n_local = x.numel()
    torch.cuda.synchronize()

    acc = xsum.Accumulator(dev)
    tot = xsum.Accumulator(dev) if world > 1 else None
    stream = torch.cuda.current_stream(dev)
    K = args.steps
    # one result record per timed step (no extra stream operation between the steps): every
    # step's bits and flags are checked after the region, not only the last one's
    res_rows = torch.zeros((max(K, 1), xsum.RESULT_BYTES), dtype=torch.uint8, device=dev)
    # multi-GPU exchange: the fused one-launch step over NVLink peer memory (symmetric memory),
    # or, if the peer buffers cannot be set up on this machine, local sum + NCCL all-gather +
    # merge_round
    pe, exchange = None, None
    if world > 1 and not seg and not args.no_fused and args.dist_backend == "nccl":
        try:
            pe = dist.PeerExchange(dev)
            exchange = "fused: one launch per rank, NVLink P2P state exchange (xsum_sum_allreduce)"
        except Exception as e:  # noqa: BLE001
            exchange = f"NCCL all-gather of 384-B states + xsum_merge_round (peer buffers unavailable: {e!r:.120})"
        if pe is not None:
            why = fused_check(xsum, dist, pe, x, acc, tot)
            if why:
                pe = None
                exchange = f"NCCL all-gather of 384-B states + xsum_merge_round (fused exchange rejected: {why})"
    elif world > 1 and not seg:
        exchange = f"{args.dist_backend} all-gather of 384-B states + xsum_merge_round"

    condsens = cfg.get("op") == "condsens"
    if condsens:
        cs_work = torch.empty(xsum.condsens_work_bytes(x.numel()), dtype=torch.uint8, device=dev)
        cs_info = torch.empty(xsum.CONDSENS_INFO_BYTES, dtype=torch.uint8, device=dev)

    def step(i=0):
        out = res_rows[i]
        if condsens:
            xsum.sum_condsens(x, 1, work=cs_work, res=out, info=cs_info)
        elif csr is not None:
            return xsum.sum_segments_csr(x, csr)[0]
        elif cfg.get("op") == "dim0":
            return xsum.exact_sum_dim(x.view(cfg["shape"]), 0)
        elif seg:
            return xsum.sum_segments(x, cfg["seg_len"])[0]
        elif world == 1:
            acc.sum(x, out=out)                          # one fused launch
        elif pe is not None:
            pe.sum(x, acc, out=out)                      # one fused launch incl. the cross-GPU merge
        else:
            dist.exact_sum_distributed(x, acc, tot, out=out)   # 2 launches + one NCCL all-gather

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    # inputs smaller than 256 MiB (c1) would be served from the 126 MB L2 on every step after
    # the first: flush L2 by writing a 256 MiB buffer before each timed step (outside its events)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if x.numel() * x.element_size() < (256 << 20) \
        else None

    def timed_region():
        res_rows.zero_()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        l0 = xsum.launch_count()
        # an event at every step boundary (per-step median / min / max); with L2 flushes the flush
        # sits between a step's end event and the next step's start event
        with ClockSampler(local_rank) as clk:
            # ~0.1 ms of device-side delay ahead of the first start event, so the host enqueues the
            # first steps while the stream is still busy: the region then holds device work only,
            # not the host's launch latency for step 0 (a 0.48 ms first step among 0.388 ms ones on c5)
            if hasattr(torch.cuda, "_sleep"):
                torch.cuda._sleep(200_000)
            for i in range(K):
                if flush is not None:
                    flush.zero_()
                if flush is not None or i == 0:
                    ev[i][0].record(stream)
                step(i)
                ev[i][1].record(stream)
            torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        return ev, clk, xsum.launch_count() - l0

    def step_ms(ev):
        out = []
        for i in range(K):
            a = ev[i][0] if (flush is not None or i == 0) else ev[i - 1][1]
            out.append(a.elapsed_time(ev[i][1]))
        return out

    ev, clk, launches = timed_region()
    # a region that saw a hardware / thermal slowdown, or SM clocks far below max with no reason
    # (a leftover clock lock), is rejected and measured once more (every rank agrees)
    first_clocks = None
    bad = torch.tensor([1.0 if clocks_rejected(clk.summary()) else 0.0], dtype=torch.float64, device=dev)
    if world > 1:
        allreduce_(bad, torch.distributed.ReduceOp.MAX)
    if float(bad.item()):
        first_clocks = clk.summary()
        ev, clk, launches = timed_region()
    # every timed step's result: identical bits on every step and rank, no peer timeout in ANY
    # step; a fused region that fails this is re-timed on the NCCL path
    fused_rejected = None
    if not seg:
        why = steps_verdict(xsum, res_rows.cpu().numpy(), world, dev)
        if why and pe is not None:
            fused_rejected = why
            pe = None
            exchange = f"NCCL all-gather of 384-B states + xsum_merge_round (fused step re-timed after: {why})"
            for _ in range(max(3, args.warmup)):
                step()
            ev, clk, launches = timed_region()
            why = steps_verdict(xsum, res_rows.cpu().numpy(), world, dev)
        if why:
            raise RuntimeError(f"timed steps invalid: {why}")
    per_step = step_ms(ev)
    # span of the K steps; with L2 flushes in between, the sum of the steps' own times
    total_ms = sum(per_step) if flush is not None else ev[0][0].elapsed_time(ev[-1][1])
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        allreduce_(t, torch.distributed.ReduceOp.MAX)
    total_ms = float(t.item())
    n_all = n_local * world
    value = n_all * K / (total_ms / 1e3)

    # dominant kernel: the accumulate launch. N=1: the step is exactly that one launch, so its
    # average duration is the span / K (launch gaps included). N>1: the fused step's local part,
    # i.e. the same kernel without the exchange (xsum_sum on the shard, one launch), timed with
    # events on its stream; exchange_us = step - local part.
    scaling = None
    if world == 1 or seg:
        kern_ms = total_ms / K
    else:
        nk = 10
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        acc.sum(x)
        a_ev.record(stream)
        for _ in range(nk):
            acc.sum(x)
        b_ev.record(stream)
        torch.cuda.synchronize()
        kern_ms = a_ev.elapsed_time(b_ev) / nk
        km = torch.tensor([kern_ms], dtype=torch.float64, device=dev)
        allreduce_(km, torch.distributed.ReduceOp.MAX)
        local_max = float(km.item())
        step_avg = total_ms / K
        scaling = {"local_sum_ms": local_max, "step_ms": step_avg,
                   "exchange_us": 1e3 * (step_avg - local_max),
                   "efficiency_est": local_max / step_avg,
                   "note": "efficiency_est = t_local / t_step, i.e. t_1 / (p t_p) with t_1 estimated as p x this "
                           "GPU count's slowest local shard scan (the scan is HBM-bound, linear in n); the driver "
                           "computes the measured efficiency from its own per-N runs"}
    peak, peak_src = measured_peak_hbm()
    esz = x.element_size()                                   # algorithmic bytes per summand
    cs_line = None
    passes = 1
    if condsens:
        # every iteration that ran reads the input once (K12 passes over the doubles; the exact pass)
        inf = xsum.CondSensInfo.from_bytes(cs_info.cpu().numpy().tobytes())
        passes = inf.iterations
        cs_line = {"r": inf.r, "iterations": inf.iterations, "exact": inf.exact, "e_cut": inf.e_cut,
                   "root_entries": len(inf.root), "rule": inf.rule}
    alg_bytes = esz * n_local * passes                      # algorithmic bytes per launch
    achieved = alg_bytes / (kern_ms / 1e3) / 1e9
    # context for the roofline: a pure streaming read of the same input in the same run (the
    # best read-only probe configuration of profiles/r01_microbench.txt: 296 blocks x 512 threads,
    # 8 x 16-B loads in flight per thread), untimed by the step
    try:
        probe_gbs = synth.probe_read_gbs(x, 1, 2 * torch.cuda.get_device_properties(dev).multi_processor_count,
                                         512, reps=10)
    except Exception:  # noqa: BLE001
        probe_gbs = None

    # context: the same step back to back for a few seconds, after the timed region (the board's
    # power cap engages after ~0.1 s; profiles/r01_sustained_power.txt)
    sustained = None
    if world == 1 and args.sustained_s > 0 and flush is None:      # (an L2-resident input would mislead)
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k_s = max(1, int(args.sustained_s / max(total_ms / K / 1e3, 1e-6)))
        with ClockSampler(local_rank, period_s=0.01) as clk_s:
            a_ev.record(stream)
            for _ in range(k_s):
                step()
            b_ev.record(stream)
            torch.cuda.synchronize()
        ms_s = a_ev.elapsed_time(b_ev)
        cs = clk_s.summary()
        sus_gbs = esz * n_local * k_s / (ms_s / 1e3) / 1e9
        sustained = {"value": n_local * k_s / (ms_s / 1e3), "unit": unit, "steps": k_s, "seconds": ms_s / 1e3,
                     "achieved_gbs": sus_gbs, "frac": sus_gbs / peak,
                     "sm_mhz": cs.get("sm_mhz"), "reasons": cs.get("reasons"),
                     "note": "context only (value is the timed region's): the same step back to back; "
                             "the 1000 W cap lowers SM clocks after ~0.1 s; frac against the same peak as roofline"}

    e2e = None
    if not args.no_e2e and condsens:
        e2e = measure_e2e_condsens(xsum, torch, x, args.e2e_steps, dev, unit, cs_work, cs_info)
    elif not args.no_e2e and not seg:
        if world == 1:
            e2e = measure_e2e(xsum, torch, x, args.e2e_steps, dev, unit,
                              want_bits=xsum.Result.from_bytes(res_rows[K - 1].cpu().numpy().tobytes()).bits)
        else:
            e2e = measure_e2e_multi(xsum, torch, dist, x, args.e2e_steps, dev, pe, acc, tot, world)
    # the timed step's exact result (the state the last step left), for the record
    result = None
    if not seg:
        import hashlib
        r_gpu = xsum.Result.from_bytes(res_rows[K - 1].cpu().numpy().tobytes())
        _, canon_gpu = acc.exact() if world == 1 else (None, None)
        result = {"value_hex": f"{r_gpu.bits:016x}", "flags": r_gpu.flags, "count": r_gpu.count}
        if canon_gpu is not None:
            result["image_sha256"] = hashlib.sha256(np.asarray(canon_gpu, dtype="<u8").tobytes()).hexdigest()
        if world == 1:
            result["sig53_exp2"] = [r_gpu.sig53, r_gpu.exp2]
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle                      # the cpu_baseline leg (test infrastructure)
        rate, cores, m, o_passes, dt, gen_name, ref = oracle_rate(args.config)
        what = "every segment of" if seg else "elements [0, %d) of" % m
        cpu = {"value": rate, "unit": unit, "cores": cores, "kind": "oracle",
               "sample": f"{what} {gen_name} ({m} elements) summed {o_passes}x by the oracle in {dt:.2f} s "
                         f"on {cores} host threads = {dt * cores:.1f} CPU-s ({cpu_model()})"}
        if seg:
            # the oracle's per-segment roundings vs the GPU's outputs of the same step, all of them
            gpu_vals = step().reshape(-1).cpu().numpy().view(np.uint64)
            cpu["matches_gpu"] = bool(gpu_vals.size == ref[0].size and (gpu_vals == ref[0]).all())
            cpu["compared"] = f"{gpu_vals.size} binary64 segment sums, bit for bit"
            r_cpu = limbs_cpu = None
        else:
            r_cpu, limbs_cpu = ref
        st = oracle_single_thread("c2" if args.config == "c2dim0" else gen_name)
        if st is not None:
            cpu["single_thread"] = st
        if result is not None and condsens:
            # a faithful rounding, not a unique one: the timed result must be
            # one of the two binary64 neighbours of the oracle's exact sum
            cpu["faithful_gpu"] = faithful(r_gpu.value, oracle.limbs_to_int(limbs_cpu))
            if cs_line is not None and cs_line["exact"]:
                cpu["matches_gpu"] = bool(r_cpu.bits == r_gpu.bits)
        elif result is not None and gen_name == args.config:
            if m == n_local:
                # the sample is the whole workload: the oracle's exact sum vs the timed GPU result
                cpu["matches_gpu"] = bool(r_cpu.bits == r_gpu.bits and r_cpu.flags == r_gpu.flags and
                                          (np.asarray(limbs_cpu) == np.asarray(canon_gpu)).all())
            elif cfg["kind"] != "bits" and m < n_local:
                # the sample is a prefix of the workload: the same prefix summed on the GPU
                rs, cs_ = xsum.Accumulator(dev).sum(x[:m], canon=True)
                rs = xsum.Result.from_bytes(rs.cpu().numpy().tobytes())
                cpu["matches_gpu_on_sample"] = bool(rs.bits == r_cpu.bits and rs.flags == r_cpu.flags and
                                                    (cs_.cpu().numpy().view(np.uint64) ==
                                                     np.asarray(limbs_cpu)).all())
    if rank == 0:
        cfg_out = {"workload": wl["desc"], "n_per_gpu": n_local, "n_total": n_all,
                   "parallelism": f"dp{world}" if world > 1 else "single",
                   "l2": ("L2 flushed (256 MiB write) before every timed step; steps timed individually"
                          if flush is not None else
                          f"inputs {x.numel() * x.element_size() / 2**30:.2f} GiB per GPU > 126 MB L2 (no flush needed)"),
                   "step": ("xsum_sum_segments_csr" if csr is not None else "xsum_sum_segments" if seg else
                            "xsum_sum fused launch" if world == 1 else exchange)}
        if fused_rejected:
            cfg_out["fused_rejected"] = fused_rejected
        line = {
            "metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": K,
            "warmup": max(3, args.warmup), "ms_per_step": total_ms / K, "higher_is_better": True,
            "scaling": wl["scaling"], "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": cfg_out,
            "step_times": dict(step_stats(per_step), note="this rank's device time per timed step (CUDA events at "
                                                          "every step boundary)"),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": profiled_traffic(args.config),
                         "kernel": {"c2f32": "k_accumulate_f32b", "c2f16": "k_accumulate_h16",
                                    "c2bf16": "k_accumulate_h16", "c5": "k_segments_halfz",
                                    "c5csr": "k_segments", "c5s16": "k_segments_lanes64s",
                                    "c2dim0": "k_sum_strided_sk", "c2cs": "xsum_sum_condsens step (all passes)",
                                    "c3cs": "xsum_sum_condsens step (all passes)"}.get(args.config, "k_accumulate"),
                         "kernel_ms": kern_ms, "algorithmic_bytes_per_launch": alg_bytes,
                         "peak_source": peak_src, "read_probe_gbs": probe_gbs,
                         "frac_of_read_probe": (achieved / probe_gbs) if probe_gbs else None,
                         # SURVEY.md §8(d)'s denominator of record: the 8 TB/s nominal HBM3e figure
                         "nominal_gbs": 8000.0, "frac_of_nominal": achieved / 8000.0,
                         "sustained_frac": sustained["frac"] if sustained else None,
                         **({"note": "the condition-number-sensitive step is ALU-bound, not HBM-bound: its r = 2 "
                                     "tree kernel keeps the ALU pipe ~88% busy (ncu, profiles/"
                                     "r02_c2cs_k_cs_tree.txt); achieved counts one input read per "
                                     "iteration that ran"} if condsens else {})},
            "clocks": dict(clk.summary(), **({"remeasured_after": first_clocks} if first_clocks else {})),
            "gpu_launches": launches,
            "e2e": e2e,
            "sustained": sustained,
            "cpu_baseline": cpu,
            "result": result,
        }
        if scaling is not None:
            line["multi_gpu"] = scaling
        if cs_line is not None:
            line["condsens"] = cs_line
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def faithful(y: float, A: int) -> bool:
    """y is RD or RU of the exact sum A * 2^-1074."""
    import math
    from fractions import Fraction
    if math.isinf(y) or math.isnan(y):
        return False
    S = Fraction(A, 1 << 1074)
    fy = Fraction(y)
    if fy == S:
        return True
    if fy < S:
        nxt = math.nextafter(y, math.inf)
        return math.isinf(nxt) or Fraction(nxt) > S
    prv = math.nextafter(y, -math.inf)
    return math.isinf(prv) or Fraction(prv) < S


def oracle_single_thread(gen_name: str, m: int = 1 << 24):
    """The oracle's single-thread rate on a 2^24-element prefix."""
    import numpy as np

    import oracle
    import synth
    cfg = synth.CONFIGS[gen_name]
    if cfg.get("fmt") is not None:
        return None
    m = min(m, cfg["n"])
    x = synth.host_generate(gen_name, 0, m)
    oracle.exact_sum(x[:4096], nthreads=1)
    t0 = time.perf_counter()
    oracle.exact_sum(x, nthreads=1)
    dt = time.perf_counter() - t0
    del x
    return {"value": m / dt, "cores": 1, "sample": f"{gen_name} elements [0, {m}) once on one thread ({dt:.2f} s)"}


def measure_e2e(xsum, torch, x_dev, steps: int, dev, unit: str = UNIT, want_bits: int | None = None):
    """Same metric through the C-ABI with a HOST buffer: per step the pinned-host -> device copy
    of the whole input (overlapped chunk by chunk, xsum_accumulate_host), the sum, the rounding
    and the 48-byte device -> host read of the result. The host copy of the input is pinned once
    (64 GiB for c4; the box has ~196 GB of host memory), outside the timed steps."""
    n = x_dev.numel()
    t0 = time.perf_counter()
    host = torch.empty(n, dtype=x_dev.dtype, pin_memory=True)
    host.copy_(x_dev)
    setup_s = time.perf_counter() - t0
    acc = xsum.Accumulator(dev)
    out = torch.empty(xsum.RESULT_BYTES, dtype=torch.uint8, pin_memory=True)

    def one():
        acc.reset().add_host(host, stage_bytes=256 << 20)
        res, _ = acc.finalize_async()
        out.copy_(res)          # synchronous D2H of the result
        return out

    one()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    got = xsum.Result.from_bytes(out.numpy().tobytes())
    del host
    line = {"value": n / dt, "unit": unit, "h2d_bytes_per_step": x_dev.element_size() * n,
            "d2h_bytes_per_step": xsum.RESULT_BYTES, "steps": steps,
            "ms_per_step": dt * 1e3, "h2d_gbs": x_dev.element_size() * n / dt / 1e9,
            "setup_s": setup_s, "api": "xsum_reset + xsum_accumulate_host + xsum_finalize_round + D2H",
            "timing": "host wall clock around the steps, after torch.cuda.synchronize"}
    if want_bits is not None:
        line["matches_device_result"] = got.bits == want_bits
    return line


def measure_e2e_condsens(xsum, torch, x_dev, steps: int, dev, unit, work, info):
    """e2e for the condition-number-sensitive workloads: per step the pinned-host -> device copy of
    the input, xsum_sum_condsens and the 48-byte result read back (host wall clock)."""
    n = x_dev.numel()
    host = torch.empty(n, dtype=x_dev.dtype, pin_memory=True)
    host.copy_(x_dev)
    buf = torch.empty_like(x_dev)
    out = torch.empty(xsum.RESULT_BYTES, dtype=torch.uint8, pin_memory=True)
    res = torch.empty(xsum.RESULT_BYTES, dtype=torch.uint8, device=dev)

    def one():
        buf.copy_(host, non_blocking=True)
        xsum.sum_condsens(buf, 1, work=work, res=res, info=info)
        out.copy_(res)

    one()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    return {"value": n / dt, "unit": unit, "h2d_bytes_per_step": x_dev.element_size() * n,
            "d2h_bytes_per_step": xsum.RESULT_BYTES, "steps": steps, "ms_per_step": dt * 1e3,
            "api": "pinned H2D copy + xsum_sum_condsens + D2H of the result"}


def allreduce_(t, op):
    """In-place all-reduce of a small CUDA tensor (host-staged for gloo process groups)."""
    import torch
    import torch.distributed as tdist
    if tdist.get_backend() == "gloo":
        h = t.cpu()
        tdist.all_reduce(h, op=op)
        t.copy_(h)
    else:
        tdist.all_reduce(t, op=op)
    return t


def fused_check(xsum, dist, pe, x, acc, tot) -> str | None:
    """Before timing the fused multi-GPU step, run it once on a 2^20-element prefix and compare
    with the NCCL all-gather + merge path on the same prefix; every rank must see bit-identical
    results and no peer timeout, else (all ranks agree on it) the NCCL path is timed instead.
    Returns None when the fused step is accepted, else the reason."""
    import torch

    probe = x[: min(x.numel(), 1 << 20)]
    res, _ = pe.sum(probe, acc)
    fused = xsum.Result.from_bytes(res.cpu().numpy().tobytes())
    ref = xsum.Result.from_bytes(dist.exact_sum_distributed(probe, xsum.Accumulator(x.device), tot)
                                 .cpu().numpy().tobytes())
    ok = fused.bits == ref.bits and fused.flags == ref.flags and not fused.flags & xsum.F_PEER_TIMEOUT
    flag = torch.tensor([1 if ok else 0], dtype=torch.int64, device=x.device)
    allreduce_(flag, torch.distributed.ReduceOp.MIN)
    if int(flag.item()):
        return None
    return (f"rank result {fused.bits:016x}/{fused.flags:#x} vs NCCL path {ref.bits:016x}/{ref.flags:#x}"
            if not ok else "another rank disagreed")


def measure_e2e_multi(xsum, torch, dist, x_dev, steps: int, dev, pe, acc, tot, world: int):
    """N > 1: per step every rank copies its shard from pinned host memory to the device, runs
    the multi-GPU step (fused or NCCL, as timed above) and reads the 48-byte result back;
    device-synchronised wall time per step, max over ranks."""
    n = x_dev.numel()
    host = torch.empty(n, dtype=torch.float64, pin_memory=True)
    host.copy_(x_dev)
    buf = torch.empty_like(x_dev)
    out = torch.empty(xsum.RESULT_BYTES, dtype=torch.uint8, pin_memory=True)

    def one():
        buf.copy_(host, non_blocking=True)
        if pe is not None:
            res, _ = pe.sum(buf, acc)
        else:
            res = dist.exact_sum_distributed(buf, acc, tot)
        out.copy_(res)
        return out

    one()
    torch.cuda.synchronize()
    torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    torch.cuda.synchronize()
    dt = torch.tensor([(time.perf_counter() - t0) / steps], dtype=torch.float64, device=dev)
    allreduce_(dt, torch.distributed.ReduceOp.MAX)
    dt = float(dt.item())
    return {"value": n * world / dt, "unit": UNIT, "h2d_bytes_per_step": 8 * n * world,
            "d2h_bytes_per_step": xsum.RESULT_BYTES * world, "ms_per_step": dt * 1e3,
            "api": "per rank: pinned H2D of the shard + multi-GPU step + D2H of the result"}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus and world == 1 and args.gpus > 1:
        print(json.dumps({"error": "run N>1 under torchrun"}))
        return 2
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)
    return 0


if __name__ == "__main__":
    sys.exit(main())
