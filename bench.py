#!/usr/bin/env python
"""Benchmark: UTF-16 repair input GB/s and % of the HBM roofline (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

Default workload (N=1 and every N, weak scaling): **config 4** — the
configuration BASELINE.json's metric ("copy & in-place ... at 1/2/4/8 GPU")
is quoted on: 2^32 units (8 GiB) per GPU, seed 4, config-0 content plus
runs of up to 1 Mi D800 and alternating H/L runs, adversarial patterns on
every shard edge. Both modes run in one invocation: the headline `value` is
copy mode; in place is reported under `modes.inplace` with its own timing,
roofline and e2e. Under torchrun each rank holds a contiguous 2^32-unit shard
of one logical N*2^32-unit buffer; the one-unit halos are read from the
neighbours' HBM over CUDA-IPC peer memory inside the single repair launch
(`--halo nccl`: an NCCL all-gather overlapped with the interior tiles).

One step = one pass of the repair path over this rank's shard. Timing: W
untimed warm-up steps, then K timed steps between a barrier +
cudaDeviceSynchronize on both sides; each step is bracketed by CUDA events on
the launching stream; value = units of all ranks x K / (max over ranks of the
summed step times). Before every step L2 is flushed by streaming-reading a
512 MiB scratch buffer (the inputs are 64x L2 anyway), and the in-place
buffer is restored from the pristine input — both outside the event pair.
stdout: ONE JSON line from rank 0.

--impl reference: the reference's own CPU implementation (oracle/_ref, built
from /root/reference/proj/src: to_well_formed with the reference's default
kernel) on all host threads over contiguous shards with exact edge fix-ups
(harness extension), on the SAME full config (both modes, same `config`
dict), rank 0 only.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "UTF-16 repair input GB/s (copy & in-place), % of HBM roofline, at 1/2/4/8 GPU"
UNIT = "GB/s"

CONFIGS = {
    # name: (cfg id, units per GPU, modes (first = headline), seed, description)
    "c0": (0, 1 << 24, ("copy",), 0,
           "config 0: copy, 2^24 units/GPU, mixed text (70% ASCII, 5% pairs, 1% lone), seed 0"),
    "c1": (1, 1 << 28, ("inplace",), 1, "config 1: in place, 2^28 units/GPU, uniform 16-bit, seed 1"),
    "c2": (2, 1 << 29, ("copy",), 2,
           "config 2: copy, 2^29 units/GPU, 50% emoji pairs + boundary straddles, seed 2"),
    "c3": (3, 1 << 20, ("batched",), 3,
           "config 3: batched copy, 2^20 strings/GPU, log-uniform 1-4095 units, seed 3"),
    "c4": (4, 1 << 32, ("copy", "inplace"), 4,
           "config 4: copy and in place, 2^32 units/GPU, config-0 mix + 1M-unit runs + shard-edge patterns, seed 4"),
    "c4copy": (4, 1 << 32, ("copy",), 4,
               "config 4: copy, 2^32 units/GPU, config-0 mix + 1M-unit runs + shard-edge patterns, seed 4"),
    "c4i": (4, 1 << 32, ("inplace",), 4,
            "config 4: in place, 2^32 units/GPU, config-0 mix + 1M-unit runs + shard-edge patterns, seed 4"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def config_dict(name: str, units_per_gpu: int, world: int) -> dict:
    """The workload description — identical in both arms (driver same_config)."""
    cfg, _per_gpu, modes, seed, desc = CONFIGS[name]
    return {"workload": desc, "config_id": cfg, "units_per_gpu": units_per_gpu, "modes": list(modes),
            "headline_mode": modes[0], "seed": seed, "parallelism": f"shard{world}" if world > 1 else "single",
            "l2": "inputs 64x L2 (8 GiB/GPU) and L2 flushed before every step (512 MiB streaming read)"
            if cfg == 4 else "L2 flushed before every step (512 MiB streaming read)"}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy_ burst)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def traffic_for(config: str, mode: str):
    """ncu DRAM bytes per launch for this config and mode, from the committed
    profile summary (profiles/traffic.json), else None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        v = d.get(f"{config}:{mode}", d.get(f"c{CONFIGS[config][0]}:{mode}"))
        return int(v) if v is not None else None
    except (OSError, ValueError, TypeError):
        return None


class ClockSampler:
    """Samples SM clock + throttle reasons via NVML while the timed region runs."""

    BAD = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml as N

            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            log("clock sampler unavailable:", e)
            self.N = None

    def _decode(self, mask: int):
        N = self.N
        names = {
            "gpu_idle": getattr(N, "nvmlClocksEventReasonGpuIdle", 0x1),
            "applications_clocks_setting": getattr(N, "nvmlClocksEventReasonApplicationsClocksSetting", 0x2),
            "sw_power_cap": getattr(N, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_slowdown": getattr(N, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sync_boost": getattr(N, "nvmlClocksEventReasonSyncBoost", 0x10),
            "sw_thermal_slowdown": getattr(N, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(N, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "hw_power_brake_slowdown": getattr(N, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        return {k for k, v in names.items() if mask & v}

    def _run(self):
        N = self.N
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                fn = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or N.nvmlDeviceGetCurrentClocksThrottleReasons
                self.reasons |= self._decode(fn(self.h)) - {"gpu_idle"}
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.N:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.N:
            self._stop.set()
            self.t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _parallel(fn, n: int, parts: int):
    """fn(a, b) over `parts` contiguous ranges of [0, n) on threads (ctypes and
    numpy copies release the GIL)."""
    bounds = [n * k // parts for k in range(parts + 1)]
    with cf.ThreadPoolExecutor(parts) as ex:
        list(ex.map(lambda k: fn(bounds[k], bounds[k + 1]), range(parts)))


def copy_mt(dst, src, threads: int | None = None):
    import numpy as np

    _parallel(lambda a, b: np.copyto(dst[a:b], src[a:b]), src.size, threads or cpu_threads())


def cpu_repair_fn(kind_pref: str = "reference", kernel_name: str | None = None):
    """(kind, fn(in_np, out_np, threads), kernel) for the reference's own code
    when oracle/_ref is built (its default kernel, or `kernel_name`), else the
    oracle port."""
    import oracle as O

    R = O.ref() if kind_pref == "reference" else None
    if R is not None:
        kname = kernel_name or O.ref_default_kernel()
        kernel = kname.encode()

        def fn(x, out, threads):
            rc = R.ref_to_well_formed_mt(O._p16(x), x.size, O._p16(out), threads, kernel)
            assert rc == 0

        return "reference", fn, kname

    def fn(x, out, threads):
        if x is out:
            tmp = O.stencil_mt(x, threads)
            copy_mt(out, tmp, threads)
        else:
            O.lib().or_stencil_mt(O._p16(x), x.size, O._p16(out), threads)

    return "port", fn, "oracle stencil"


def cpu_workload(config: str, units: int, total: int | None = None):
    """Host copy of the first `units` units of the config's data (CPU oracle
    generators, multi-threaded over independent windows)."""
    import numpy as np

    import oracle as O

    cfg, per_gpu, modes, seed, _ = CONFIGS[config]
    if cfg == 3:
        return O.gen_c3(units, seed)
    total = total or units
    x = np.empty(units, dtype=np.uint16)
    shard_len = per_gpu if cfg == 4 else 0

    def gen(a, b):
        if b > a:
            rc = O.lib().or_gen_config(cfg, seed, total, shard_len, a, b - a, O._p16(x[a:b]))
            assert rc == 0

    _parallel(gen, units, max(1, min(cpu_threads(), units >> 20 or 1)))
    return x, None


def time_cpu(config: str, units: int, mode: str, reps: int, warmup: int, budget_s: float,
             kernel_name: str | None = None, threads: int | None = None, data=None):
    """Input GB/s of the CPU repair over `units` of the config in `mode`.
    Returns the whole-run rate (units x reps / summed rep time, like the GPU
    arm's `value`) and the best rep (the reference's measure() statistic)."""
    import numpy as np

    import oracle as O

    kind, fn, kname = cpu_repair_fn(kernel_name=kernel_name)
    threads = threads or cpu_threads()
    x, offsets = data if data is not None else cpu_workload(config, units, CONFIGS[config][1])
    out = np.empty_like(x)
    times = []
    t_start = time.perf_counter()
    for i in range(warmup + reps):
        if mode == "inplace":
            copy_mt(out, x, threads)  # restore, outside the timing
            t0 = time.perf_counter()
            fn(out, out, threads)
        elif mode == "batched":
            t0 = time.perf_counter()
            # per-string repair is the reference semantics; the reference has no
            # batched API, so each string goes through fix_scalar (oracle) —
            # the threaded stencil is not valid across string edges.
            out = O.fix_batched(x, offsets)
        else:
            t0 = time.perf_counter()
            fn(x, out, threads)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
        if time.perf_counter() - t_start > budget_s and len(times) >= 1:
            break
    nbytes = 2 * x.size
    return {
        "gbps": nbytes * len(times) / sum(times) / 1e9,
        "gbps_best": nbytes / min(times) / 1e9,
        "kind": kind if mode != "batched" else "port",
        "cores": threads if mode != "batched" else 1,
        "kernel": kname if mode != "batched" else "oracle fix_scalar per string",
        "units": int(x.size),
        "reps": len(times),
        "ms_per_rep": 1e3 * sum(times) / len(times),
        "best_ns": int(min(times) * 1e9),
        "mean_ns": sum(times) / len(times) * 1e9,
    }


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg, per_gpu, modes, seed, desc = CONFIGS[args.config]
    t0 = time.perf_counter()
    data = cpu_workload(args.config, per_gpu, per_gpu)
    log(f"reference arm: generated {data[0].size} units in {time.perf_counter() - t0:.1f} s")
    res = {}
    for mode in modes:
        res[mode] = time_cpu(args.config, per_gpu, mode, reps=args.steps, warmup=args.warmup, budget_s=240.0,
                             data=data)
    head = res[modes[0]]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    sample = (f"{head['units']} units of {args.config} per rep (full config"
              + (f"; one shard's worth: the CPU rate does not depend on how the {world}-shard job is split"
                 if world > 1 else "")
              + f"), {head['reps']} timed reps after {args.warmup} warm-up; value = units x reps / summed rep time; "
              "in place restored before every rep (outside the timing)")
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(head["gbps"], 3),
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": head["reps"],
        "warmup": args.warmup,
        "ms_per_step": round(head["ms_per_rep"], 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u16",
        "data": "synthetic",
        "config": config_dict(args.config, head["units"], world),
        "modes": {m: {"value": round(r["gbps"], 3), "best_gbps": round(r["gbps_best"], 3),
                      "ms_per_step": round(r["ms_per_rep"], 3), "reps": r["reps"]} for m, r in res.items()},
        "cpu_baseline": {"value": round(head["gbps"], 3), "unit": UNIT, "cores": head["cores"],
                         "kind": head["kind"], "kernel": head["kernel"], "sample": sample},
        "e2e": {"value": round(head["gbps"], 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    if args.csv:
        write_csv(args.csv, [(f"reference-{r['kernel']}-x{r['cores']}-{m}", r["units"], [r["best_ns"]] * 1,
                              r["mean_ns"]) for m, r in res.items()])
    return 0


# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2601_06349_b200 as P
    from paper_2601_06349_b200 import _lib
    from paper_2601_06349_b200 import dist as pdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("U16M_BENCH_SHARE_GPU") == "1" or local >= torch.cuda.device_count():
        # U16M_BENCH_SHARE_GPU: code-path check of the N>1 line on a box with
        # fewer GPUs than ranks (ranks share devices; the numbers are then
        # meaningless). Otherwise: a launcher that gave every rank its own
        # CUDA_VISIBLE_DEVICES (one visible GPU, index 0); if ranks really
        # shared a GPU, NCCL refuses to initialise below.
        local %= max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    distributed = world > 1 or args.force_dist
    if distributed:
        if os.environ.get("U16M_BENCH_SHARE_GPU") == "1":
            pdist.init_process_group_for_repair("gloo")  # NCCL refuses two ranks on one GPU
        else:
            pdist.init_process_group_for_repair("nccl", device_id=dev)
    L = _lib.raw()
    cfg, per_gpu, modes, seed, desc = CONFIGS[args.config]
    if args.units:
        per_gpu = args.units
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream

    # Pinned host buffers for the e2e leg, allocated first: pinning 16 GiB
    # makes the VM's memory manager busy for seconds afterwards, and host
    # memory activity slows the PCIe DMA by up to 20 %
    # (scripts/e2e_noise_probe.py); by the time the e2e leg runs it has settled.
    e2e_note = None

    def pinned_pair(n):
        """Two pinned host buffers of n units, or None on every rank when any
        rank cannot pin them (N ranks pin N x 16 GiB on one host)."""
        nonlocal e2e_note
        try:
            bufs = (torch.empty(n, dtype=torch.int16, pin_memory=True),
                    torch.empty(n, dtype=torch.int16, pin_memory=True))
        except RuntimeError as e:
            log("pinned host allocation failed, e2e leg skipped:", e)
            bufs = None
        if distributed:
            ok = torch.tensor([1.0 if bufs is not None else 0.0], device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if ok.item() == 0.0:
                bufs = None
        if bufs is None:
            e2e_note = "e2e leg skipped: pinned host buffers could not be allocated on every rank"
            args.no_e2e = True
        return bufs

    e2e_bufs = None
    if not args.no_e2e and cfg != 3:
        e2e_bufs = pinned_pair(per_gpu)

    # ---- data (device-side generators; inputs resident in HBM) ----
    offsets = None
    if cfg == 3:
        data, offsets = _lib.gen_c3(per_gpu, seed=seed + 1000 * rank, device=dev)
        units = data.numel()
    else:
        units = per_gpu
        data = _lib.gen_config(cfg, units * world, seed=seed, first=rank * units, count=units,
                               shard_len=units if cfg == 4 else 0, device=dev)
    if cfg == 3 and not args.no_e2e:  # the batch's length is known only now (still ahead of the timing)
        e2e_bufs = pinned_pair(units)
    # `data` stays pristine; copy mode writes `work`, in place restores `work`
    # from `data` before every step and repairs it.
    work = torch.empty_like(data)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    flush.fill_(1)
    torch.cuda.synchronize()

    halos = {}
    if distributed and cfg != 3 and args.halo == "ipc":
        try:
            halos["copy"] = pdist.PeerHalo(data)      # neighbours' pristine shards
            halos["inplace"] = pdist.PeerHalo(work)   # neighbours' in-place buffers
        except Exception as e:  # noqa: BLE001
            log("PeerHalo (CUDA IPC) setup failed, using the NCCL gather:", e)
            halos = {}

    def step_kernel(mode):
        if mode == "batched":
            _lib._check(L.u16m_to_well_formed_batched_n(data.data_ptr(), data.numel(), offsets.data_ptr(),
                                                       offsets.numel() - 1, work.data_ptr(), sptr))
        elif mode in halos:
            halos[mode].repair(work if mode == "copy" else None)
        elif distributed:
            pdist.repair_shard(data if mode == "copy" else work, work, all_nonempty=True)
        elif mode == "inplace":
            _lib._check(L.u16m_to_well_formed_in_place(work.data_ptr(), units, sptr))
        else:
            _lib._check(L.u16m_to_well_formed(data.data_ptr(), units, work.data_ptr(), sptr))

    def prepare(mode):
        if mode == "inplace":
            work.copy_(data)
        if not args.warm:
            _lib.l2_flush(flush)

    results = {}
    clk_all = []
    for mode in modes:
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        for _ in range(args.warmup):
            prepare(mode)
            step_kernel(mode)
        torch.cuda.synchronize()
        if distributed:
            dist.barrier()
        torch.cuda.synchronize()
        launches0 = P.launch_count()
        repair_launches = 0
        with ClockSampler(local) as clk:
            wall0 = time.perf_counter()
            for i in range(args.steps):
                prepare(mode)
                ev[i][0].record(stream)
                c0 = P.launch_count()
                step_kernel(mode)
                repair_launches += P.launch_count() - c0
                ev[i][1].record(stream)
            torch.cuda.synchronize()
            if distributed:
                dist.barrier()
            torch.cuda.synchronize()
            wall = time.perf_counter() - wall0
        clk_all.append(clk.summary())
        step_ms = [a.elapsed_time(b) for a, b in ev]
        t = torch.tensor([sum(step_ms) / 1e3, min(step_ms) / 1e3], dtype=torch.float64, device=dev)
        if distributed:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        # correctness spot check of the last step (cheap, device-side): the
        # repaired buffer is well-formed (batched: every string is, and none
        # ends with a high or starts with a low surrogate, so the whole buffer is)
        ok = P.count_unpaired(work) == 0
        results[mode] = {"t_max": float(t[0].item()), "best_max": float(t[1].item()), "t_local": sum(step_ms) / 1e3,
                         "step_ms": step_ms, "launches": repair_launches,
                         "launches_incl_flush": P.launch_count() - launches0, "wall": wall, "ok": bool(ok)}

    in_bytes = 2 * units
    extra = 8 * offsets.numel() if offsets is not None else 0
    peak, peak_src = peaks()

    def mode_summary(mode):
        r = results[mode]
        value = world * in_bytes * args.steps / r["t_max"] / 1e9
        # at N=1 (and under the IPC halo at any N) a step is exactly one repair
        # launch, so the step time is the kernel's launch duration
        single = not distributed or mode in halos or mode == "batched"
        kernel_s = r["t_local"] / args.steps
        algo = 4 * units + extra
        achieved = algo / kernel_s / 1e9
        tr = traffic_for(args.config, mode)
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": tr,
                "algorithmic_bytes_per_launch": algo, "peak_source": peak_src,
                "kernel_ms": round(kernel_s * 1e3, 4),
                "step_is_one_launch": single}
        if tr:
            # in place writes back only the 32-byte sectors holding a rewrite,
            # so the algorithmic frac can exceed 1; this is the DRAM-level one
            roof["dram_gbs_from_traffic"] = round(tr / kernel_s / 1e9, 1)
            roof["dram_frac_from_traffic"] = round(tr / kernel_s / 1e9 / peak, 4)
        if extra:
            roof["frac_without_offsets"] = round(4 * units / kernel_s / 1e9 / peak, 4)
        return value, {"value": round(value, 3), "ms_per_step": round(r["t_max"] * 1e3 / args.steps, 4),
                       "best_ms": round(r["best_max"] * 1e3, 4), "roofline": roof,
                       "gpu_launches": r["launches"], "gpu_launches_incl_flush": r["launches_incl_flush"],
                       "output_check_well_formed": r["ok"], "wall_s_timed_loop": round(r["wall"], 4)}

    summaries = {m: mode_summary(m) for m in modes}

    # ---- e2e through the reference-facing C-ABI with host (pinned) buffers ----
    e2e = {}
    if not args.no_e2e and cfg != 3:
        multi = world == 1 and torch.cuda.device_count() > 1 and hasattr(L, "u16m_to_well_formed_host_multi")
        hin, hout = e2e_bufs
        hin.copy_(data)
        e2e_steps = max(3, min(args.steps, args.e2e_steps))
        def e2e_call(mode):
            if mode == "inplace":
                # Restore the host buffer by DMA from the pristine device
                # copy, outside the timed region: the input arrives as if
                # from a storage/network DMA (a CPU memcpy right before the
                # call leaves dirty lines the H2D DMA then competes with).
                hout.copy_(data)
                torch.cuda.synchronize()
            src, dst = (hout, hout) if mode == "inplace" else (hin, hout)
            if distributed:
                dist.barrier()
            t0 = time.perf_counter()
            if multi:
                _lib._check(L.u16m_to_well_formed_host_multi(src.data_ptr(), units, dst.data_ptr(), 0, None))
            else:
                _lib._check(L.u16m_to_well_formed_host(src.data_ptr(), units, dst.data_ptr()))
            return time.perf_counter() - t0

        for mode in modes:
            # Untimed warm-up until the host-memory system is steady: three
            # consecutive calls within 3 % of each other (at least 2, at most
            # 20 calls; every rank decides on the max over ranks). This VM
            # slows PCIe DMA by 10-20 % for seconds after a process frees or
            # touches tens of GiB of memory (profiles/r02/e2e_noise.txt) — e.g.
            # the reference arm that runs right before this one.
            warm = []
            while True:
                warm.append(e2e_call(mode))
                last = warm[-3:]
                steady = len(warm) >= 3 and max(last) <= 1.03 * min(last)
                if distributed:
                    flag = torch.tensor([0.0 if steady else 1.0], device=dev)
                    dist.all_reduce(flag, op=dist.ReduceOp.MAX)
                    steady = flag.item() == 0.0
                if (steady and len(warm) >= 2) or len(warm) >= 20:
                    break
            times = [e2e_call(mode) for _ in range(e2e_steps)]
            te = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
            if distributed:
                dist.all_reduce(te, op=dist.ReduceOp.MAX)
            # spot check: the host result equals the device result of the same mode
            ok = bool(torch.equal(hout[: 1 << 20].to(dev), work[: 1 << 20])) and \
                bool(torch.equal(hout[-(1 << 20):].to(dev), work[-(1 << 20):]))
            e2e[mode] = {"value": round(world * in_bytes * len(times) / float(te.item()) / 1e9, 3), "unit": UNIT,
                         "h2d_bytes_per_step": in_bytes, "d2h_bytes_per_step": in_bytes,
                         "api": ("u16m_to_well_formed_host_multi (all visible GPUs)" if multi else
                                 "u16m_to_well_formed_host") + " — the C ABI behind utf16mend::to_well_formed"
                                " on host spans; pinned host buffers",
                         "host_input": ("restored by device-to-host DMA before each step (outside the timing)"
                                        if mode == "inplace" else "written once"),
                         "steps": len(times), "matches_device_result": ok,
                         "step_gbps": [round(in_bytes / t / 1e9, 1) for t in times],
                         "warmup_calls": len(warm),
                         "warmup_rule": "untimed calls until 3 consecutive agree within 3 % (2-20 calls)"}
        del hin, hout, e2e_bufs
    elif not args.no_e2e and cfg == 3:
        # the batched form on host memory (the C ABI behind the C++ batched API on host spans)
        hin, hout = e2e_bufs
        hin.copy_(data)
        hoff = offsets.cpu()
        nstr = offsets.numel() - 1
        e2e_steps = max(3, min(args.steps, args.e2e_steps))
        times = []
        for i in range(2 + e2e_steps):
            if distributed:
                dist.barrier()
            t0 = time.perf_counter()
            _lib._check(L.u16m_to_well_formed_batched_host(hin.data_ptr(), units, hoff.data_ptr(), nstr,
                                                           hout.data_ptr()))
            dt = time.perf_counter() - t0
            if i >= 2:
                times.append(dt)
        te = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
        if distributed:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        ok = bool(torch.equal(hout[: 1 << 20].to(dev), work[: 1 << 20])) and \
            bool(torch.equal(hout[-(1 << 20):].to(dev), work[-(1 << 20):]))
        e2e["batched"] = {"value": round(world * in_bytes * len(times) / float(te.item()) / 1e9, 3), "unit": UNIT,
                          "h2d_bytes_per_step": in_bytes + extra, "d2h_bytes_per_step": in_bytes,
                          "api": "u16m_to_well_formed_batched_host — the C ABI behind the C++ batched API on host "
                                 "spans; pinned host buffers, host offsets",
                          "host_input": "written once", "steps": len(times), "matches_device_result": ok,
                          "step_gbps": [round(in_bytes / t / 1e9, 1) for t in times]}
        del hin, hout, e2e_bufs

    cpu = cpu_row = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            mode0 = modes[0]
            cpu_units = min(units, 1 << 27) if cfg != 3 else min(per_gpu, 1 << 16)
            sample = cpu_workload(args.config, cpu_units, CONFIGS[args.config][1])
            # a bounded sample: ~10 s of CPU work (reps until the budget is spent)
            r = time_cpu(args.config, cpu_units, mode0, reps=100000, warmup=1, budget_s=10.0, data=sample)
            cpu_row = (f"reference-{r['kernel']}-x{r['cores']}-{mode0}", r["units"], [r["best_ns"]], r["mean_ns"])
            cpu = {"value": round(r["gbps"], 3), "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
                   "best_gbps": round(r["gbps_best"], 3),
                   "sample": f"first {r['units']} units of {args.config} in {mode0} mode ({r['kernel']}), "
                             f"{r['reps']} reps in ~10 s, input restored before every in-place rep"}
            # The reference's scalar and SIMD paths, 1 thread (its own
            # methodology, bench.hpp:51) and all threads (harness extension).
            if r["kind"] == "reference" and cfg != 3:
                paths = {}
                small = (sample[0][: 1 << 24], None)
                for kname in ("scalar", r["kernel"]):
                    for th in (1, cpu_threads()):
                        q = time_cpu(args.config, 0, mode0, reps=100000, warmup=1, budget_s=2.0, kernel_name=kname,
                                     threads=th, data=sample if th > 1 else small)
                        paths[f"{kname}_{th}thr"] = round(q["gbps_best"], 3)
                cpu["paths_gbps_best"] = paths
        except Exception as e:  # noqa: BLE001
            log("cpu baseline failed:", e)

    if distributed:
        # release the neighbours' IPC mappings before any producer exits
        used_ipc = bool(halos)
        halos.clear()
        torch.cuda.synchronize()
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return 0
    head = modes[0]
    value, head_sum = summaries[head]
    clocks = {"sm_mhz": statistics.median([c["sm_mhz"] for c in clk_all if c["sm_mhz"]] or [0]) or None,
              "sm_max_mhz": clk_all[0]["sm_max_mhz"],
              "reasons": sorted(set().union(*[set(c["reasons"]) for c in clk_all])),
              "samples": sum(c["samples"] for c in clk_all)}
    line = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": head_sum["ms_per_step"],
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u16",
        "data": "synthetic",
        "config": config_dict(args.config, units, world) if not args.units else
        {**config_dict(args.config, units, world), "workload": desc + f" (REDUCED: {units} units/GPU)"},
        "run": {"halo": ((("ipc-peer-loads" if used_ipc else "nccl-allgather")) if distributed else None),
                "warm": bool(args.warm)},
        "roofline": head_sum["roofline"],
        "modes": {m: {**s, **({"e2e": e2e[m]} if m in e2e else {})} for m, (_, s) in summaries.items()},
        "cpu_baseline": cpu,
        "e2e": e2e.get(head) or {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                                 "note": e2e_note or "e2e leg skipped (--no-e2e)"},
        "gpu_launches": head_sum["gpu_launches"],
        "gpu_launches_all_modes": sum(s["gpu_launches"] for _, s in summaries.values()),
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    if args.csv:
        rows = []
        for m in modes:
            r = results[m]
            rows.append((f"cuda-sm100a{'-x' + str(world) if world > 1 else ''}-{m}", world * units,
                         [int(x * 1e6) for x in r["step_ms"]], None))
        if cpu_row:
            rows.append(cpu_row)
        write_csv(args.csv, rows)
    return 0


CSV_HEADER = "impl,input_units,bytes,best_ns,mean_ns,gbps,error_margin_pct"


def csv_row(impl: str, units: int, best_ns: int, mean_ns: float) -> str:
    """One row of the reference's CSV report (proj/src/bench.cpp:151-163):
    best_ns = fastest step (integer ns), mean_ns = mean step, gbps = decimal
    GB/s of input bytes (2 B/unit) over the best step, error_margin_pct =
    100 (mean - best) / best (bench.cpp:77-87). Numbers round-trip exactly
    through the reference's parse_csv (%.17g, bench.cpp:159)."""
    best_ns = max(1, int(best_ns))
    nbytes = 2 * units
    gbps = nbytes / best_ns
    margin = 100.0 * (mean_ns - best_ns) / best_ns
    return f"{impl},{units},{nbytes},{best_ns},{mean_ns!r},{gbps!r},{margin!r}"


def write_csv(path, rows):
    """Append rows (impl, units, step_ns list, mean_ns|None) in the reference
    schema; the header is written when the file is new."""
    new = not os.path.exists(path)
    with open(path, "a") as f:
        if new:
            f.write(CSV_HEADER + "\n")
        for impl, units, steps_ns, mean_ns in rows:
            best = min(steps_ns)
            mean = float(mean_ns) if mean_ns is not None else sum(steps_ns) / len(steps_ns)
            f.write(csv_row(impl, units, best, mean) + "\n")


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--units", type=int, default=0,
                    help="override units per GPU (probes only; the line is then labelled REDUCED)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10, help="timed e2e steps per mode (at most --steps)")
    ap.add_argument("--warm", action="store_true",
                    help="skip the L2 flush between steps (warm-cache number, SURVEY.md §8(d) C0; never the headline)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the sharded step even at N=1 (under torchrun)")
    ap.add_argument("--halo", default="ipc", choices=["ipc", "nccl"],
                    help="N>1 halo exchange: neighbour units read over CUDA IPC peer memory inside the one "
                         "repair kernel (default), or an NCCL all-gather overlapped with the interior tiles")
    ap.add_argument("--csv", default=None,
                    help="also append rows in the reference bench CSV schema (proj/src/bench.cpp:151-163)")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (timing rules)")
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
