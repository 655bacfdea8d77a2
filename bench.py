#!/usr/bin/env python
"""Benchmark: UTF-16 repair input GB/s and % of the HBM roofline (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1] [--impl ours|reference]

One step = one pass of the repair path over this rank's shard of one
synthetic BASELINE config, inputs resident in HBM. Default workload (N=1 and
every N, weak scaling): config 1 — in place, 2^28 uniform-random 16-bit units
per GPU (512 MiB), seed 1 — the configuration BASELINE.json's metric is
quoted on that fits one GPU. Under torchrun each rank holds a contiguous
2^28-unit shard of one logical N·2^28-unit buffer; the 2-unit halo exchange
(NCCL all-gather) is inside the step.

Timing: W untimed warm-up steps, then K timed steps between a barrier +
cudaDeviceSynchronize on both sides. In-place repair destroys its input, so
before every step the shard is restored from a pristine copy and L2 is flushed
by streaming-reading a 512 MiB scratch buffer (both outside the CUDA-event
pair that brackets each step); the reported time is the sum of the K
event-timed steps, max over ranks. stdout: ONE JSON line from rank 0.

--impl reference: the reference's own CPU implementation (oracle/_ref, built
from /root/reference/proj/src: to_well_formed with the reference's default
kernel), on all host threads over contiguous shards with exact edge fix-ups
(harness extension), on the same config; rank 0 only.
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

METRIC = "UTF-16 repair input GB/s (copy & in-place), % of HBM roofline, at 1/2/4/8 GPU"
UNIT = "GB/s"

CONFIGS = {
    # name: (cfg id, units per GPU, mode, seed, description)
    "c0": (0, 1 << 24, "copy", 0, "config 0: copy, 2^24 units/GPU, mixed text (70% ASCII, 5% pairs, 1% lone), seed 0"),
    "c1": (1, 1 << 28, "inplace", 1, "config 1: in place, 2^28 units/GPU, uniform 16-bit, seed 1"),
    "c2": (2, 1 << 29, "copy", 2, "config 2: copy, 2^29 units/GPU, 50% emoji pairs + boundary straddles, seed 2"),
    "c3": (3, 1 << 20, "batched", 3, "config 3: batched copy, 2^20 strings/GPU, log-uniform 1-4095 units, seed 3"),
    "c4": (4, 1 << 32, "copy", 4, "config 4: copy, 2^32 units/GPU, config-0 mix + 1M-unit runs + shard-edge patterns, seed 4"),
    "c4i": (4, 1 << 32, "inplace", 4, "config 4: in place, 2^32 units/GPU, config-0 mix + runs + shard-edge patterns, seed 4"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy_ burst)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def traffic_for(config: str):
    """ncu DRAM bytes per launch for this config, from the committed profile
    summary (profiles/traffic.json), else None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            v = json.load(f).get(config)
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
            time.sleep(0.005)

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


def cpu_repair_fn(kind_pref: str = "reference", kernel_name: str | None = None):
    """(kind, fn(in_np, out_np, threads)) for the reference's own code when
    oracle/_ref is built (its default kernel, or `kernel_name`), else the
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
            out[:] = tmp
        else:
            O.lib().or_stencil_mt(O._p16(x), x.size, O._p16(out), threads)

    return "port", fn, "oracle stencil"


def cpu_workload(config: str, units: int):
    """Host copy of the config's data (CPU oracle generators)."""
    import oracle as O

    cfg, per_gpu, mode, seed, _ = CONFIGS[config]
    if cfg == 3:
        data, offsets = O.gen_c3(units, seed)
        return data, offsets
    return O.gen_config(cfg, units, seed=seed, shard_len=units if cfg == 4 else 0), None


def time_cpu(config: str, units: int, reps: int, warmup: int, budget_s: float, kernel_name: str | None = None,
             threads: int | None = None):
    """Best/mean input GB/s of the CPU repair over `units` of the config."""
    import numpy as np

    import oracle as O

    kind, fn, kname = cpu_repair_fn(kernel_name=kernel_name)
    threads = threads or cpu_threads()
    x, offsets = cpu_workload(config, units)
    mode = CONFIGS[config][2]
    out = np.empty_like(x)
    times = []
    t_start = time.perf_counter()
    for i in range(warmup + reps):
        if mode == "inplace":
            out[:] = x
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
    best = min(times)
    return {
        "gbps_best": nbytes / best / 1e9,
        "gbps_mean": nbytes / (sum(times) / len(times)) / 1e9,
        "kind": kind if mode != "batched" else "port",
        "cores": threads if mode != "batched" else 1,
        "kernel": kname if mode != "batched" else "oracle fix_scalar per string",
        "units": int(x.size),
        "reps": len(times),
        "ms_per_rep": 1e3 * sum(times) / len(times),
    }


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg, per_gpu, mode, seed, desc = CONFIGS[args.config]
    units = per_gpu if cfg != 4 else min(per_gpu, 1 << 28)
    r = time_cpu(args.config, units, reps=args.steps, warmup=args.warmup, budget_s=150.0)
    sample = (f"{r['units']} units of {args.config} per rep ({'full config' if units == per_gpu else 'bounded sample'})"
              f", {r['reps']} timed reps after {args.warmup} warm-up, best rep")
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(r["gbps_best"], 3),
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": r["reps"],
        "warmup": args.warmup,
        "ms_per_step": round(r["ms_per_rep"], 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u16",
        "data": "synthetic",
        "config": {"workload": desc, "units": r["units"], "mode": mode,
                   "kernel": r["kernel"], "threads": r["cores"]},
        "cpu_baseline": {"value": round(r["gbps_best"], 3), "unit": UNIT, "cores": r["cores"],
                         "kind": r["kind"], "sample": sample},
        "e2e": {"value": round(r["gbps_best"], 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2601_06349_b200 as P
    from paper_2601_06349_b200 import _lib
    from paper_2601_06349_b200 import dist as pdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    distributed = world > 1 or args.force_dist
    if distributed:
        pdist.init_process_group_for_repair("nccl", device_id=dev)
    L = _lib.raw()
    cfg, per_gpu, mode, seed, desc = CONFIGS[args.config]
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream

    # ---- data (device-side generators; inputs resident in HBM) ----
    offsets = None
    if cfg == 3:
        data, offsets = _lib.gen_c3(per_gpu, seed=seed + 1000 * rank, device=dev)
        units = data.numel()
    else:
        units = per_gpu
        total = units * world
        data = _lib.gen_config(cfg, total, seed=seed, first=rank * units, count=units,
                               shard_len=units if cfg == 4 else 0, device=dev)
    pristine = data.clone() if mode == "inplace" else None
    out = torch.empty_like(data) if mode != "inplace" else data
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    flush.fill_(1)
    torch.cuda.synchronize()

    halo = None
    if distributed and mode != "batched" and args.halo == "ipc":
        try:
            halo = pdist.PeerHalo(data)
        except Exception as e:  # noqa: BLE001
            log("PeerHalo (CUDA IPC) setup failed, using the NCCL gather:", e)
            halo = None

    def step_kernel():
        if mode == "batched":
            _lib._check(L.u16m_to_well_formed_batched_n(data.data_ptr(), data.numel(), offsets.data_ptr(),
                                                       offsets.numel() - 1, out.data_ptr(), sptr))
        elif halo is not None:
            halo.repair(out)
        elif distributed:
            pdist.repair_shard(data, out)
        elif mode == "inplace":
            _lib._check(L.u16m_to_well_formed_in_place(data.data_ptr(), units, sptr))
        else:
            _lib._check(L.u16m_to_well_formed(data.data_ptr(), units, out.data_ptr(), sptr))

    def prepare():
        if pristine is not None:
            data.copy_(pristine)
        if not args.warm:
            _lib.l2_flush(flush)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    for _ in range(args.warmup):
        prepare()
        step_kernel()
    torch.cuda.synchronize()
    graph = None
    launches_per_step = None
    if distributed and args.graph:
        # Optional: the sharded step (interior kernel + side-stream gather +
        # edge kernel) captured once into a CUDA graph and replayed.
        prepare()
        torch.cuda.synchronize()
        c0 = P.launch_count()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step_kernel()
        launches_per_step = P.launch_count() - c0
        for _ in range(2):
            prepare()
            graph.replay()
        torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = P.launch_count()
    repair_launches = 0
    with ClockSampler(local) as clk:
        wall0 = time.perf_counter()
        for i in range(args.steps):
            prepare()
            ev[i][0].record(stream)
            c0 = P.launch_count()
            if graph is not None:
                graph.replay()
                repair_launches += launches_per_step
            else:
                step_kernel()
                repair_launches += P.launch_count() - c0
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        if distributed:
            dist.barrier()
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_local = sum(step_ms) / 1e3
    t = torch.tensor([t_local], dtype=torch.float64, device=dev)
    if distributed:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    all_launches = P.launch_count() - launches0

    # correctness spot check of the last step against the first repair (cheap, device-side)
    # (batched: every repaired string is well-formed and none ends with a high
    # or starts with a low surrogate, so the concatenation — config 3's whole
    # buffer — is well-formed too)
    ok = P.count_unpaired(out) == 0

    in_bytes = 2 * units
    extra = 8 * offsets.numel() if offsets is not None else 0
    value = world * in_bytes * args.steps / t_max / 1e9
    peak, peak_src = peaks()
    kernel_s = t_local / args.steps  # at N=1 the step is exactly one kernel launch
    algo_bytes = 4 * units + extra
    achieved = algo_bytes / kernel_s / 1e9

    # ---- e2e through the reference-facing C-ABI with host (pinned) buffers ----
    e2e = None
    if not args.no_e2e and mode != "batched":
        hin = torch.empty(units, dtype=torch.int16, pin_memory=True)
        hin.copy_(pristine if pristine is not None else data)
        hout = hin if mode == "inplace" else torch.empty_like(hin).pin_memory()
        e2e_steps = max(3, min(args.steps, 20))
        times = []
        for i in range(args.warmup + e2e_steps):
            if mode == "inplace":
                # Restore the host input by DMA from the pristine device copy,
                # outside the timed region: the input arrives as if from a
                # storage/network DMA. A CPU memcpy restore instead leaves
                # hundreds of MB of dirty lines / pending write-backs in the
                # host memory system that the H2D DMA then competes with
                # (39 vs 46 GB/s measured by scripts/e2e_timeline_probe.py).
                hin.copy_(pristine)
                torch.cuda.synchronize()
            if distributed:
                dist.barrier()
            t0 = time.perf_counter()
            _lib._check(L.u16m_to_well_formed_host(hin.data_ptr(), units, hout.data_ptr()))
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                times.append(dt)
        te = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
        if distributed:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": round(world * in_bytes * len(times) / float(te.item()) / 1e9, 3), "unit": UNIT,
               "h2d_bytes_per_step": in_bytes, "d2h_bytes_per_step": in_bytes,
               "api": "u16m_to_well_formed_host (C ABI behind utf16mend::to_well_formed), pinned host buffers",
               "host_input": ("restored by device-to-host DMA before each step (outside the timing)"
                              if mode == "inplace" else "written once"),
               "steps": len(times)}
    elif mode == "batched" and not args.no_e2e:
        e2e = {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
               "note": "batched host path not timed"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu_units = min(units, 1 << 26) if cfg != 3 else min(per_gpu, 1 << 16)
            # a bounded sample: ~10 s of CPU work (reps until the budget is spent)
            r = time_cpu(args.config, cpu_units, reps=100000, warmup=1, budget_s=10.0)
            cpu = {"value": round(r["gbps_best"], 3), "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
                   "sample": f"first {r['units']} units of {args.config} ({r['kernel']}), best of {r['reps']} reps "
                             f"in ~10 s, input restored before every in-place rep"}
            # The reference's scalar and SIMD paths, 1 thread (its own
            # methodology, bench.hpp:51) and all threads (harness extension).
            if r["kind"] == "reference" and mode != "batched":
                paths = {}
                for kname in ("scalar", r["kernel"]):
                    for th in (1, cpu_threads()):
                        q = time_cpu(args.config, cpu_units if th > 1 else min(cpu_units, 1 << 24), reps=100000,
                                     warmup=1, budget_s=2.0, kernel_name=kname, threads=th)
                        paths[f"{kname}_{th}thr"] = round(q["gbps_best"], 3)
                cpu["paths_gbps"] = paths
        except Exception as e:  # noqa: BLE001
            log("cpu baseline failed:", e)

    if distributed:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return 0
    line = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(t_max * 1e3 / args.steps, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u16",
        "data": "synthetic",
        "config": {"workload": desc, "units_per_gpu": units, "mode": mode,
                   "parallelism": f"shard{world}" if distributed else "single",
                   "halo": (("ipc-peer-loads" if halo is not None else "nccl-allgather") if distributed else None),
                   "l2": ("WARM: no L2 flush between steps (labelled warm number, not the headline)" if args.warm else
                          "flushed before every step (512 MiB streaming read) + restore outside the event pair"),
                   "hbm_fraction_of_measured_peak": round((value / world) * (algo_bytes / in_bytes) / peak, 4),
                   "output_check_well_formed": bool(ok)},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic_for(args.config),
                     # in place writes back only sectors holding a rewrite, so the
                     # algorithmic frac can exceed 1; this is the DRAM-level one
                     "dram_gbs_from_traffic": (round(traffic_for(args.config) / kernel_s / 1e9, 1)
                                               if traffic_for(args.config) and world == 1 else None),
                     "dram_frac_from_traffic": (round(traffic_for(args.config) / kernel_s / 1e9 / peak, 4)
                                                if traffic_for(args.config) and world == 1 else None),
                     "algorithmic_bytes_per_launch": algo_bytes, "peak_source": peak_src,
                     **({"frac_without_offsets": round(4 * units / kernel_s / 1e9 / peak, 4)} if extra else {}),
                     "kernel_ms": round(kernel_s * 1e3, 4)},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": repair_launches,
        "gpu_launches_incl_flush": all_launches,
        "clocks": clk.summary(),
        "wall_s_timed_loop": round(wall, 4),
    }
    print(json.dumps(line), flush=True)
    if args.csv:
        write_csv(args.csv, [("cuda-sm100a" + (f"-x{world}" if world > 1 else ""), world * units, t_max / args.steps,
                              None)] + ([("reference-" + cpu["kind"], None, None, cpu)] if cpu else []))
    return 0


def write_csv(path, rows):
    """Append rows in the reference's CSV schema (proj/src/bench.cpp:151-163):
    impl,input_units,bytes,best_ns,mean_ns,gbps,error_margin_pct (decimal GB/s
    of input bytes, 2 B per unit)."""
    header = "impl,input_units,bytes,best_ns,mean_ns,gbps,error_margin_pct"
    new = not os.path.exists(path)
    with open(path, "a") as f:
        if new:
            f.write(header + "\n")
        for impl, units, sec, cpu in rows:
            if cpu is not None:
                gbps = cpu["value"]
                f.write(f"{impl},,,,,{gbps:.3f},\n")
            else:
                ns = sec * 1e9
                f.write(f"{impl},{units},{2 * units},{ns:.0f},{ns:.0f},{2 * units / ns:.3f},0.000\n")


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c1", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--warm", action="store_true",
                    help="skip the L2 flush between steps (warm-cache number, SURVEY.md §8(d) C0; never the headline)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the sharded (NCCL halo exchange) step even at N=1 (under torchrun)")
    ap.add_argument("--halo", default="ipc", choices=["ipc", "nccl"],
                    help="N>1 halo exchange: neighbour units read over CUDA IPC peer memory inside the one "
                         "repair kernel (default), or an NCCL all-gather overlapped with the interior tiles")
    ap.add_argument("--graph", action="store_true",
                    help="capture the sharded step in a CUDA graph (measured: no gain at N=1, 0.136 vs 0.133 ms)")
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
