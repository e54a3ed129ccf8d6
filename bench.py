"""Benchmark: semisort Grecords/s on BASELINE.json's headline config.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c5|c3|c4|c1|graph] [--scaling weak|strong] [--mode eq|lt]

Workloads:
  c2 (default, the metric's config, BASELINE.json configs[1]): semisort of
     10^9 (uint64 key, uint64 value) records per GPU; keys Zipf(s=1.2) ranks
     over [1, 10^9] hashed to 64 bits (key = mix64(rank - 1)), value =
     global record index.
  c5 (configs[4], the multi-GPU config): 50/50 mix of uniform 64-bit keys
     and Zipf(0.8) ranks over [1, 10^8] (minus 1), value = global index;
     weak (10^9 per GPU) or strong (8 x 10^9 in total) scaling.
  c3 / c4: collect_reduce(summing64) / histogram on one GPU (configs[2], [3]).
  c1 (configs[0]): the reference's CPU-runnable 2^20 case; call latency,
     the reference package timed on the same input, byte-compared.
  graph: CSR transpose.
Inputs are synthetic, seeded and generated on the device (same families,
parameters and sampler as the reference generator).

N > 1: `bench.py --gpus N` started without WORLD_SIZE re-launches itself
under torch.distributed.run (one process per GPU, NCCL); under torchrun it
runs directly.  Each rank hash-partitions its shard, ONE all-to-allv of
packed records moves them, and the local semisort runs from the received
buffer (paper_2304_10078_b200.distributed).  `value` = records of all ranks
/ the max over ranks of the step time.

Timing: W untimed warm-up steps, then K steps; before every step the input
is restored from a pristine device copy (or regenerated under strong
scaling): a >= 16 GB write that flushes the 126 MB L2.  Then barrier +
synchronize, CUDA events around the library call only (the reference
protocol, cli.py:94-109), synchronize + barrier, max over ranks.  `e2e`
repeats the step through the public API from pinned host buffers with the
H2D input copy and the D2H result copy inside the timed region.
`cpu_baseline` / `--impl reference`: the reference package itself
(baseline/_ref, `workers = os.cpu_count()`) on a bounded sample of the same
workload on this host; the numpy restatement (oracle/) when the reference
is not installed.  The output of the last timed step is validated outside
the timed region (`validated`).
"""

from __future__ import annotations

import argparse
import contextlib
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_DEFAULT = 10**9
ZIPF_S = 1.2
UNIVERSE = 10**9
C5_S, C5_UNIVERSE, C5_TOTAL = 0.8, 10**8, 8 * 10**9
B_ALG = 72          # K + 4R bytes / record (semisort, 8 B keys, 16 B records)
NOMINAL_HBM = 8.0e12
NVLINK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md); nominal 900
U64 = (1 << 64) - 1

# generator families of ss_generate (paper_2304_10078_b200.datagen.FAMILIES)
WORKLOADS = {
    "c2": {"family": "zipfian", "param": ZIPF_S, "universe": UNIVERSE, "hash_ranks": True,
           "metric": "semisort Grecords/s (n=1e9 u64 k/v, Zipf 1.2 hashed)",
           "desc": "c2: semisort n=1e9 per GPU, uint64 key/value, Zipf s=1.2 ranks over [1,1e9] hashed (mix64), "
                   "value = global index"},
    "c5": {"family": "mix", "param": C5_S, "universe": C5_UNIVERSE, "hash_ranks": False,
           "metric": "semisort Grecords/s (u64 k/v, 50/50 uniform-64 / Zipf 0.8 over 1e8)",
           "desc": "c5: semisort, uint64 key/value, 50/50 mix of uniform [0,2^64) and Zipf s=0.8 ranks over "
                   "[1,1e8] minus 1, value = global index"},
}
FAMILY_ID = {"uniform": 0, "exponential": 1, "zipfian": 2, "uniform64": 3, "mix": 4}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons during the timed region.

    Polls NVML every 25 ms (NVML at 2 ms contended with the launches of
    small-kernel workloads), falling back to nvidia-smi when NVML is
    unavailable.  A CPU environment reports "unsampled".
    """

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4))
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int | None):
        self.index = index
        self.samples = []   # (sm_mhz, max_mhz, set of reason names)
        self._stop = threading.Event()
        self._t = None
        self._nv = self._h = None
        if index is None:
            return
        try:   # NVML set up outside the timed region
            import pynvml as nv
            nv.nvmlInit()
            self._nv, self._h = nv, nv.nvmlDeviceGetHandleByIndex(index)
            self._mx = float(nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM))
            self._reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
        except Exception:
            self._nv = None

    def _sample_nvml(self):
        nv, h = self._nv, self._h
        bits = self._reasons(h)
        self.samples.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)), self._mx,
                             {name for name, bit in self.REASONS if bits & bit}))

    def _run_smi(self):
        names = [name for name, _ in self.REASONS]
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                f = [x.strip() for x in out.split(",")]
                if len(f) >= 8 and f[0].replace(".", "").isdigit():
                    self.samples.append((float(f[0]), float(f[1]),
                                         {n for n, v in zip(names, f[4:8]) if v.lower() == "active"}))
            except Exception:
                pass
            self._stop.wait(0.05)

    def _run(self):
        if self._nv is None:
            return self._run_smi()
        while not self._stop.wait(0.025):
            try:
                self._sample_nvml()
            except Exception:
                return

    def __enter__(self):
        if self.index is None:
            return self
        if self._nv is not None:
            self._sample_nvml()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        if self._t is None:
            return
        self._stop.set()
        self._t.join(timeout=10)
        if self._nv is not None:
            try:
                self._sample_nvml()
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [x[0] for x in self.samples]
        reasons = set().union(*(x[2] for x in self.samples))
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(x[1] for x in self.samples),
                "sm_min_mhz": min(sm), "reasons": sorted(reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# environment: one process per GPU (NCCL), or CPU tensors over gloo (tests)
# ---------------------------------------------------------------------------

class Env:
    """Rank / world / device plus the collectives and the timer the bench
    orchestration needs.  CUDA: events on the current stream, NCCL
    collectives.  CPU (tests): perf_counter, gloo."""

    def __init__(self, rank: int, world: int, device, dist_on: bool):
        self.rank, self.world, self.device, self.dist_on = rank, world, device, dist_on
        self.cuda = getattr(device, "type", "cpu") == "cuda"

    def sync(self):
        if self.cuda:
            import torch
            torch.cuda.synchronize(self.device)

    def barrier(self):
        if self.dist_on:
            import torch.distributed as dist
            dist.barrier()

    def _reduce(self, vals, op, dtype):
        import torch
        import torch.distributed as dist
        t = torch.tensor(vals, dtype=dtype, device=self.device)
        if self.dist_on:
            dist.all_reduce(t, op=op)
        return t.cpu().tolist()

    def max(self, x: float) -> float:
        import torch
        import torch.distributed as dist
        return float(self._reduce([float(x)], dist.ReduceOp.MAX if self.dist_on else None, torch.float64)[0])

    def sum_u64(self, vals):
        """Sums mod 2^64 over ranks (int64 addition wraps like uint64)."""
        import torch
        import torch.distributed as dist
        signed = [v - (1 << 64) if v >= (1 << 63) else v for v in vals]
        return [v & U64 for v in self._reduce(signed, dist.ReduceOp.SUM if self.dist_on else None, torch.int64)]

    def all(self, ok: bool) -> bool:
        import torch
        import torch.distributed as dist
        return bool(self._reduce([0 if ok else 1], dist.ReduceOp.SUM if self.dist_on else None, torch.int64)[0] == 0)

    @contextlib.contextmanager
    def timed(self, out: list):
        """Appends the duration (ms) of the block: CUDA events on the current
        stream (synchronised on both sides), else the host clock."""
        if self.cuda:
            import torch
            st = torch.cuda.current_stream(self.device)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            yield
            e1.record(st)
            torch.cuda.synchronize(self.device)
            out.append(e0.elapsed_time(e1))
        else:
            t0 = time.perf_counter()
            yield
            out.append((time.perf_counter() - t0) * 1e3)


def cuda_env():
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=dev)
    return Env(rank, world, dev, world > 1)


# ---------------------------------------------------------------------------
# semisort workloads (c2, c5): the library path (DeviceHooks) behind the
# orchestration; tests substitute CPU hooks and run it over gloo
# ---------------------------------------------------------------------------

class DeviceHooks:
    """Generation, the timed library calls and the validators on the GPU."""

    def __init__(self, env: Env):
        import paper_2304_10078_b200 as S
        self.S = S
        self.env = env
        self.adapter = S.UIntKeyAdapter()

    def generate(self, w, n, first, out=None):
        import torch

        import paper_2304_10078_b200 as S
        from paper_2304_10078_b200 import _lib
        from paper_2304_10078_b200.core import _stream
        c = WORKLOADS[w]
        if out is None:
            out = S.RecordArray(torch.empty(n, dtype=torch.uint64, device=self.env.device),
                                torch.empty(n, dtype=torch.uint64, device=self.env.device))
        _lib.check(_lib.lib().ss_generate(FAMILY_ID[c["family"]], float(c["param"]), int(c["universe"]), n, first,
                                          8, 1, 1 if c["hash_ranks"] else 0, out.keys.data_ptr(),
                                          out.values.data_ptr(), 8, 1, 0, _stream(self.env.device)))
        return out

    def restore(self, src, work):
        work.keys.copy_(src.keys)
        work.values.copy_(src.values)

    def telemetry(self):
        return self.S.Telemetry(timing=True)

    def sort(self, work, mode, params, tel):
        self.S.semisort(work, self.adapter, mode, params, telemetry=tel)
        return work

    def dist_sort(self, work, mode, tel, recv_block=None, scratch=None):
        from paper_2304_10078_b200.distributed import dist_semisort
        return dist_semisort(work, self.adapter, mode, telemetry=tel, recv_block=recv_block, scratch=scratch)

    def validate_single(self, src, out):
        """Exact O(n) check (bitmap permutation, records intact, contiguity by a
        distinct-key count, stability) against the pristine input."""
        from paper_2304_10078_b200.validate import count_distinct, validate_indexed
        rep = validate_indexed(src.keys, out.keys, out.values, count_distinct(src.keys))
        return {"permutation": rep.is_permutation, "contiguous": rep.is_contiguous, "stable": rep.is_stable}

    def shard_check(self, w, out, parts, rank):
        """(bad_record, runs, bad_stable, bad_dest, sum v, sum v^2, sum mix64 v, distinct keys) of a shard."""
        import ctypes as C

        from paper_2304_10078_b200 import _lib
        from paper_2304_10078_b200.core import _stream, _workspace
        from paper_2304_10078_b200.validate import count_distinct
        c = WORKLOADS[w]
        m = len(out)
        res = (C.c_uint64 * 7)()
        ws = _workspace(4096, self.env.device)
        _lib.check(_lib.lib().ss_validate_shard(FAMILY_ID[c["family"]], float(c["param"]), int(c["universe"]), 1,
                                                1 if c["hash_ranks"] else 0, out.keys.data_ptr(),
                                                out.values.data_ptr(), m, 8, parts, rank, ws.data_ptr(), ws.numel(),
                                                res, _stream(self.env.device)))
        return [int(x) for x in res] + [count_distinct(out.keys) if m else 0]

    def index_fingerprint(self, lo, hi):
        import ctypes as C

        from paper_2304_10078_b200 import _lib
        from paper_2304_10078_b200.core import _stream, _workspace
        res = (C.c_uint64 * 3)()
        ws = _workspace(4096, self.env.device)
        _lib.check(_lib.lib().ss_index_fingerprint(lo, hi, ws.data_ptr(), ws.numel(), res, _stream(self.env.device)))
        return [int(x) for x in res]

    def heavy_stats(self, src, params):
        """Level-1 heavy keys of the input (the root's own sample, core.py:221-260)
        and the fraction of records they hold (c2 39 / 0.578)."""
        import numpy as np
        import torch

        from paper_2304_10078_b200.core import mix64_pair, sample_and_bucket
        from paper_2304_10078_b200.records import signed_view
        rng = np.random.Generator(np.random.Philox(key=mix64_pair(params.seed, 0)))
        table = sample_and_bucket(src, self.adapter, params, 0, rng)
        if not len(table):
            return {"n_heavy": 0, "heavy_fraction": 0.0}
        hk = torch.tensor([k - (1 << 64) if k >= (1 << 63) else k for k in table.keys], dtype=torch.int64,
                          device=src.keys.device)
        frac = float(torch.isin(signed_view(src.keys), hk).sum().item()) / max(len(src), 1)
        return {"n_heavy": len(table), "heavy_fraction": frac}


def _semisort_roofline(world, n_local, ms, tel, steps, peak_gbs, traffic):
    """Dominant kernel (blocked distributing) and whole-step rooflines; at
    G > 1 the step model adds the partition and the exchange."""
    dist_ms = tel.phase_ms.get("distribute", 0.0) / steps if tel is not None else 0.0
    moved = tel.bucket_assignments / steps if tel is not None else 0.0   # records scattered per step (local sort)
    achieved = (moved * 32) / (dist_ms / 1e3) / 1e9 if dist_ms > 0 else None
    g = world
    b_hbm = B_ALG + ((40 + 32 * (g - 1) / g) if g > 1 else 0)
    b_nvl = 16 * (g - 1) / g
    t = ms / 1e3
    step_gbs = b_hbm * n_local / t / 1e9
    roof_rate = min(NOMINAL_HBM / b_hbm, (NVLINK_GBS * 1e9 / b_nvl) if b_nvl else float("inf"))   # rec/s per GPU
    return ({"bound": "hbm", "kernel": "k_distribute1 (single-pass blocked distributing scatter, all levels)",
             "achieved": achieved, "peak": peak_gbs, "unit": "GB/s",
             "frac": (achieved / peak_gbs) if achieved else None, "traffic": traffic,
             "bytes_model": "32 B per bucketed record (read 16 B + write 16 B)"},
            {"bytes_per_record_hbm": b_hbm, "bytes_per_record_nvlink": b_nvl, "achieved_gbs": step_gbs,
             "peak": peak_gbs, "frac_of_measured": step_gbs / peak_gbs,
             "frac_of_nominal_8tbs": step_gbs * 1e9 / NOMINAL_HBM,
             "nvlink_gbs_per_direction": (b_nvl * n_local / t / 1e9) if b_nvl else 0.0,
             "roofline_rate_grec_per_gpu": roof_rate / 1e9,
             "frac_of_roofline": (n_local / t) / roof_rate})


def _traffic(workload):
    """Mean ncu DRAM bytes per k_distribute1 launch of one step of `workload`
    (profiles/traffic.json, one `ncu --set full` capture), or None."""
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        t = json.load(open(tpath))
        ls = t[workload]["launches"]
        return sum(x["dram_read"] + x["dram_write"] for x in ls) / len(ls), len(ls), t.get("note", "")
    except Exception:
        return None


def run_semisort(args, env: Env, hooks, emit=print):
    """c2 / c5 at N = env.world GPUs; rank 0 emits one JSON line."""
    import torch
    S = hooks.S
    w = args.workload
    world, rank = env.world, env.rank
    strong = args.scaling == "strong"
    total = args.total if strong else args.n * world
    n = total // world if strong else args.n
    first = rank * n
    if strong and world == 1 and total * 16 * 2 > 170e9:
        if rank == 0:
            emit(json.dumps({"metric": WORKLOADS[w]["metric"], "n_gpus": 1, "scaling": "strong",
                             "skipped": f"strong scaling: {total} records (input + scratch = "
                                        f"{total * 32 / 1e9:.0f} GB) do not fit one GPU"}))
        return None
    params = S.TuningParams.for_input(n)
    # buffers: strong scaling keeps TWO record buffers per rank (input/receive
    # block and send/scratch block, each with headroom) and regenerates the
    # input every step; weak scaling restores from a pristine copy
    cap = n + n // 8 + 4096
    recv_block = scratch = None
    if world > 1 and strong:
        blk = torch.empty(2 * cap, dtype=torch.uint64, device=env.device)
        scratch = torch.empty(2 * cap, dtype=torch.uint64, device=env.device)
        work = S.core._raw(blk[:n], blk[cap:cap + n], "u64")
        recv_block = blk
        src = None
    else:
        src = hooks.generate(w, n, first)
        work = src.empty_like()
        if world > 1:
            scratch = torch.empty(2 * cap, dtype=torch.uint64, device=env.device)
            recv_block = torch.empty(2 * cap, dtype=torch.uint64, device=env.device)

    def step(tel=None, times=None):
        if src is None:
            hooks.generate(w, n, first, work)
        else:
            hooks.restore(src, work)
        env.sync()
        env.barrier()
        env.sync()
        sink = times if times is not None else []
        with env.timed(sink):
            if world == 1:
                out = hooks.sort(work, args.mode, params, tel)
            else:
                out = hooks.dist_sort(work, args.mode, tel, recv_block=recv_block, scratch=scratch)
        env.barrier()
        return out

    for _ in range(args.warmup):   # same code path as the timed steps (phase events on)
        step(hooks.telemetry())
    times = []
    tel = hooks.telemetry()
    with ClockSampler(env.device.index if env.cuda else None) as clk:
        for _ in range(args.steps):
            out = step(tel, times)
    ms_local = sum(times) / len(times)
    ms = env.max(ms_local)
    value = total / (ms / 1e3) / 1e9
    peak_gbs, peak_kind = measured_peaks()
    tr = _traffic(w) if (world == 1 and args.mode == "eq" and n == N_DEFAULT) else None
    roof, step_roof = _semisort_roofline(world, n, ms, tel, args.steps, peak_gbs, tr[0] if tr else None)
    roof["peak_kind"] = peak_kind
    if tr is not None:
        launches = tr[1]
        roof["alg_bytes_per_launch"] = tel.bucket_assignments / args.steps * 32 / launches
        roof["traffic_note"] = f"mean over the step's {launches} distribute launches; " + tr[2]

    # validation of the last timed step's output (outside the timed region)
    valid, vdetail = None, None
    if not args.no_validate:
        if world == 1 and src is not None and hasattr(hooks, "validate_single"):
            vdetail = hooks.validate_single(src, out)
            ok = all(vdetail.values())
        else:
            sc = hooks.shard_check(w, out, world, rank)
            bad_rec, runs, bad_st, bad_dest, s1, s2, s3, distinct = sc
            local_ok = bad_rec == 0 and bad_st == 0 and bad_dest == 0 and runs == distinct
            cnt = env.sum_u64([len(out), s1, s2, s3])
            expect = [total] + hooks.index_fingerprint(0, total) if rank == 0 else None
            all_ok = env.all(local_ok)
            ok = all_ok and (rank != 0 or cnt == expect)
            ok = env.all(ok)
            vdetail = {"records_intact": all_ok, "contiguous_and_stable_and_dest": all_ok,
                       "fingerprints_match": (cnt == expect) if rank == 0 else None,
                       "shard_records": len(out)}
        valid = bool(ok)
    heavy = None
    if not args.no_validate and world == 1 and src is not None and hasattr(hooks, "heavy_stats") and w == "c2":
        heavy = hooks.heavy_stats(src, params)
    shard_max = env.max(float(len(out)))

    e2e = None
    if not args.no_e2e and env.cuda:
        del work
        if src is not None:
            torch.cuda.empty_cache()
        e2e = e2e_leg(args, env, hooks, src, n, first, params)
    cpu = None
    if not args.no_cpu and rank == 0 and world == 1 and w == "c2":
        cpu = cpu_baseline(args.cpu_n)
    if rank == 0:
        line = {
            "metric": (WORKLOADS[w]["metric"] if args.mode == "eq" else "semisort< (lt) " + WORKLOADS[w]["metric"]),
            "value": value, "unit": "Grecords/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "ms_steps_rank0": [round(t, 3) for t in times],
            "higher_is_better": True, "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic (device-generated, seeded)",
            "config": {"workload": WORKLOADS[w]["desc"], "n_per_gpu": n, "n_total": total,
                       "params": "TuningParams.for_input(n) (reference defaults, seed 1)",
                       "l2": ("input regenerated before each step (16 GB write flushes L2)" if src is None else
                              "input restored from a pristine copy before each step (16 GB write flushes L2)"),
                       "parallelism": f"dp{world}" if world > 1 else "single",
                       "exchange": ("one packed all_to_all_v (NCCL) of 16-byte records" if world > 1 else None),
                       "max_shard_records": int(shard_max)},
            "roofline": roof, "step_roofline": step_roof,
            "phase_ms_per_step": {k: v / args.steps for k, v in tel.phase_ms.items()},
            "levels": tel.levels / args.steps, "gpu_launches": tel.kernel_launches,
            "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu, "validated": valid,
            "validation": vdetail, "l1_heavy": heavy,
        }
        emit(json.dumps(line))
        return line
    return None


def e2e_leg(args, env, hooks, src, n, first, params):
    """The same step through the public API from pinned host memory: H2D of
    the inputs and D2H of the result inside the timed region (never fails the
    bench line: an error is reported in the e2e object instead)."""
    import torch
    S = hooks.S
    try:
        en = args.e2e_n or (n if env.world == 1 else min(n, 250_000_000))
        if src is None:
            src = hooks.generate(args.workload, en, first)
        hk = torch.empty(en, dtype=torch.uint64, pin_memory=True)
        hv = torch.empty(en, dtype=torch.uint64, pin_memory=True)
        cap = en + en // 4 + 4096
        ok = torch.empty(cap, dtype=torch.uint64, pin_memory=True)
        ov = torch.empty(cap, dtype=torch.uint64, pin_memory=True)
        hk.copy_(src.keys[:en])
        hv.copy_(src.values[:en])
        del src
        torch.cuda.empty_cache()
        p_e = S.TuningParams.for_input(en)
        ts, moved = [], 0
        for i in range(max(1, min(args.steps, 3)) + 1):
            env.sync()
            env.barrier()
            sink = ts if i else []
            with env.timed(sink):
                data = S.RecordArray(hk, hv)                     # H2D through the public API
                if env.world == 1:
                    S.semisort(data, hooks.adapter, args.mode, p_e)
                    res = data
                else:
                    from paper_2304_10078_b200.distributed import dist_semisort
                    res = dist_semisort(data, hooks.adapter, args.mode)
                m = len(res)
                if m > cap:
                    raise RuntimeError("received shard larger than the pinned output buffer")
                ok[:m].copy_(res.keys, non_blocking=True)       # D2H of the result
                ov[:m].copy_(res.values, non_blocking=True)
            env.barrier()
            moved = m
            del data, res
        e_ms = env.max(sum(ts) / len(ts))
        tot = en * env.world
        return {"value": tot / (e_ms / 1e3) / 1e9, "unit": "Grecords/s", "h2d_bytes_per_step": 16 * tot,
                "d2h_bytes_per_step": 16 * tot, "ms_per_step": e_ms, "n": tot,
                "path": ("RecordArray(pinned host tensors) -> semisort -> copy to pinned host" if env.world == 1 else
                         "per rank: RecordArray(pinned host shard) -> dist_semisort (NCCL) -> output shard to pinned "
                         f"host; max over ranks; bytes summed over ranks (rank 0 moved {moved} records out)")}
    except Exception as exc:
        return {"error": f"{type(exc).__name__}: {exc}"[:300]}


# ---------------------------------------------------------------------------
# CPU baselines: the reference package itself (baseline/_ref), else the port
# ---------------------------------------------------------------------------

REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _reference_module():
    """The unmodified reference package installed into baseline/_ref (pip
    --target), or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "semisort")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import semisort as R   # noqa: N812
        if os.path.dirname(os.path.dirname(os.path.abspath(R.__file__))) != REF_DIR:
            return None
        return R
    except Exception:
        return None


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _ref_c2_input(R, n):
    """The first n records of the reference's own c2 dataset: its generator's
    per-block Philox streams and rejection-inversion Zipf sampler
    (datagen.py:66-108) over the 1e9-rank universe, key = mix64(rank - 1),
    value = index."""
    import numpy as np
    from semisort import datagen, hashing
    spec = datagen.DistributionSpec("zipfian", ZIPF_S, UNIVERSE, 64, seed=1)
    ranks = np.empty(n, dtype=np.uint64)
    for b in range(-(-n // datagen.GEN_BLOCK)):
        lo, hi = b * datagen.GEN_BLOCK, min((b + 1) * datagen.GEN_BLOCK, n)
        ranks[lo:hi] = datagen._zipf_block(datagen._block_rng(spec, b), hi - lo, ZIPF_S, UNIVERSE)
    return hashing.mix64_array(ranks - np.uint64(1)), np.arange(n, dtype=np.uint64)


def reference_semisort_rate(n, steps, warmup):
    """(Grec/s, seconds per step, description) of the reference's semisort on n
    records of c2 with all host cores, or None when it is not installed."""
    R = _reference_module()
    if R is None:
        return None
    keys, vals = _ref_c2_input(R, n)
    base = R.RecordArray(keys, vals)
    params = R.TuningParams.for_input(n)
    workers = os.cpu_count() or 1
    times = []
    for i in range(warmup + steps):
        work = base.copy()
        t0 = time.perf_counter()
        R.semisort(work, R.UIntKeyAdapter(), "eq", params, workers=workers)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    t = statistics.median(times)
    return n / t / 1e9, t, (f"reference package semisort (baseline/_ref, unmodified; semisort(..., workers={workers}))"
                            f" on the first {n} records of the c2 dataset (its own generator, 1e9-rank Zipf 1.2, "
                            f"hashed), value = index; median of {steps} after {warmup} warm-up; host "
                            f"{_cpu_model()}"), workers


def cpu_baseline(n_sample: int):
    """The reference CPU path on a bounded sample (reference package, all
    cores; the oracle port single-threaded when the package is absent)."""
    r = reference_semisort_rate(min(n_sample, 1 << 24), 1, 1)
    if r is not None:
        v, t, desc, workers = r
        return {"value": v, "unit": "Grecords/s", "cores": workers, "kind": "reference", "sample": desc}
    import numpy as np

    import oracle as O
    from oracle.datagen import gen_keys_values
    ranks, _ = gen_keys_values("zipfian", ZIPF_S, n_sample, 64, seed=1, universe=UNIVERSE)
    keys = O.mix64_np(ranks - np.uint64(1))
    vals = np.arange(n_sample, dtype=np.uint64)
    P = O.OracleParams.derive(n_sample)
    t0 = time.perf_counter()
    O.semisort(keys, vals, P)
    t = time.perf_counter() - t0
    return {"value": n_sample / t / 1e9, "unit": "Grecords/s", "cores": 1, "kind": "port",
            "sample": f"semisort of {n_sample} records, Zipf s=1.2 ranks over [1, 1e9] hashed, value=index; "
                      f"reference algorithm restated in numpy (oracle/), single thread, {t:.2f} s"}


def reference_arm(args):
    """--impl reference: the reference's CPU semisort (baseline/_ref, all host
    cores) on a bounded sample of c2 per step; rank 0 only."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    steps, warmup = max(args.steps, 1), max(args.warmup, 0)
    # size the sample so the whole run stays within ~2-3 minutes
    n = args.ref_n
    if n is None:
        probe = reference_semisort_rate(1 << 20, 1, 0)
        rate = probe[0] * 1e9 if probe else 2e6
        budget = 150.0 / (steps + warmup)
        n = 1 << max(18, min(24, int(math.log2(max(rate * budget, 1)))))
    r = reference_semisort_rate(n, steps, warmup)
    if r is not None:
        v, t, desc, workers = r
        kind = "reference"
    else:   # the numpy restatement, single thread
        import numpy as np

        import oracle as O
        from oracle.datagen import gen_keys_values
        ranks, _ = gen_keys_values("zipfian", ZIPF_S, n, 64, seed=1, universe=UNIVERSE)
        keys = O.mix64_np(ranks - np.uint64(1))
        vals = np.arange(n, dtype=np.uint64)
        P = O.OracleParams.derive(n)
        for _ in range(warmup):
            O.semisort(keys, vals, P)
        t0 = time.perf_counter()
        for _ in range(steps):
            O.semisort(keys, vals, P)
        t = (time.perf_counter() - t0) / steps
        v, workers, kind = n / t / 1e9, 1, "port"
        desc = f"{n} records per step, numpy restatement of the reference algorithm (oracle/), single thread"
    line = {"metric": WORKLOADS["c2"]["metric"], "value": v, "unit": "Grecords/s",
            "n_gpus": args.gpus, "steps": steps, "warmup": warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": f"c2 semisort sample n={n} (bounded CPU sample of the 1e9 workload)",
                       "key": "Zipf(1.2) rank over [1, 1e9] -> mix64(rank-1)", "value": "index"},
            "cpu_baseline": {"value": v, "unit": "Grecords/s", "cores": workers, "kind": kind, "sample": desc},
            "e2e": {"value": v, "unit": "Grecords/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# aggregation workloads (c3, c4) and the graph app, one GPU
# ---------------------------------------------------------------------------

AGG = {   # the aggregation configs (not the headline metric)
    "c3": {"metric": "collect_reduce sum64 Grecords/s (n=1e9 u64 k/v, exponential 1e-4)", "family": "exponential",
           "param": 1e-4, "key_bits": 64, "values": "random", "shift": 32, "kind": "sum64", "b_alg": 56.0,
           "desc": "c3: collect_reduce(summing64), n=1e9, keys floor(Exponential(scale 1e4)) u64, "
                   "values uniform u64 >> 32"},
    "c4": {"metric": "histogram Grecords/s (n=1e9 u32, uniform [0,1e7))", "family": "uniform", "param": 1e7,
           "key_bits": 32, "values": "none", "shift": 0, "kind": "count", "b_alg": 16.12,
           "desc": "c4: histogram, n=1e9 u32 keys uniform [0, 1e7), no values"},
}


def agg_cpu_baseline(w, n_sample):
    """The reference package's collect_reduce / histogram (baseline/_ref, all
    cores) on a bounded sample; the oracle port when it is absent."""
    import numpy as np
    c = AGG[w]
    R = _reference_module()
    if R is not None:
        from semisort import datagen
        g = datagen.generate(datagen.DistributionSpec(c["family"], c["param"], n_sample, c["key_bits"], seed=1))
        vals = (g.values >> np.uint64(c["shift"])) if c["values"] != "none" else None
        data = R.RecordArray(g.keys, vals)
        spec = R.ReduceSpec.summing64() if c["kind"] == "sum64" else R.ReduceSpec.counting()
        workers = os.cpu_count() or 1
        t0 = time.perf_counter()
        R.collect_reduce(data, R.UIntKeyAdapter(), spec, R.TuningParams.for_input(n_sample), workers=workers)
        t = time.perf_counter() - t0
        return {"value": n_sample / t / 1e9, "unit": "Grecords/s", "cores": workers, "kind": "reference",
                "sample": f"reference package collect_reduce (baseline/_ref, workers={workers}) on "
                          f"{n_sample} records of {c['desc'].split(',')[0]} (its own generator, seed 1), {t:.2f} s; "
                          f"host {_cpu_model()}"}
    import oracle as O
    from oracle.datagen import gen_keys_values
    keys, vals = gen_keys_values(c["family"], c["param"], n_sample, c["key_bits"], seed=1)
    vals = (vals.astype(np.uint64) >> np.uint64(c["shift"])) if c["values"] != "none" else None
    P = O.OracleParams.derive(n_sample)
    t0 = time.perf_counter()
    O.collect_reduce(keys, vals, P, c["kind"])
    t = time.perf_counter() - t0
    return {"value": n_sample / t / 1e9, "unit": "Grecords/s", "cores": 1, "kind": "port",
            "sample": f"{c['desc'].split(',')[0]} on {n_sample} records (same families, seed 1); reference "
                      f"algorithm restated in numpy (oracle/), single thread, {t:.2f} s"}


def agg_validate(src, res, kind):
    """Independent device reduction (torch): c4 bincount, c3 sort + segmented
    sum; compared per key with the library's pairs (multiset order)."""
    import torch

    from paper_2304_10078_b200.records import signed_view
    keys = signed_view(src.keys).to(torch.int64)
    if src.keys.dtype == torch.uint32:
        keys = keys & 0xFFFFFFFF
    rk = signed_view(res.key_tensor).to(torch.int64)
    if res.key_tensor.dtype == torch.uint32:
        rk = rk & 0xFFFFFFFF
    ra = signed_view(res.agg_tensor)
    order = torch.argsort(rk)
    rk, ra = rk[order], ra[order]
    if kind == "count" and int(keys.max().item()) < (1 << 28):
        cnt = torch.bincount(keys, minlength=int(keys.max().item()) + 1)
        ek = torch.nonzero(cnt).flatten()
        ea = cnt[ek]
    else:
        sk, idx = torch.sort(keys)
        ek, counts = torch.unique_consecutive(sk, return_counts=True)
        if kind == "count":
            ea = counts
        else:
            v = signed_view(src.values)[idx]
            cs = torch.cumsum(v, 0)            # int64 wraps like the uint64 sum
            ends = torch.cumsum(counts, 0) - 1
            ea = cs[ends]
            ea[1:] = ea[1:] - cs[ends[:-1]]
            del v, cs
        del sk, idx
    return bool(ek.numel() == rk.numel() and torch.equal(ek, rk) and torch.equal(ea.to(torch.int64), ra))


def agg_main(args):
    """--workload c3|c4: collect_reduce / histogram on one GPU (same JSON contract)."""
    import torch

    import paper_2304_10078_b200 as S
    from paper_2304_10078_b200.datagen import generate_device
    w = args.workload
    c = AGG[w]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    env = Env(0, 1, dev, False)
    n = args.n
    src = generate_device(c["family"], c["param"], n, key_bits=c["key_bits"], seed=1, values=c["values"],
                          value_shift=c["shift"], device=dev)
    adp = S.UIntKeyAdapter()
    spec = S.ReduceSpec.summing64() if c["kind"] == "sum64" else S.ReduceSpec.counting()
    params = S.TuningParams.for_input(n)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # 256 MB > L2, written before every step

    def one(tel=None, times=None):
        flush.fill_(1)
        env.sync()
        with env.timed(times if times is not None else []):
            res = S.collect_reduce(src, adp, spec, params, telemetry=tel)
        return res

    for _ in range(args.warmup):   # same code path as the timed steps (phase events on)
        one(S.Telemetry(timing=True))
    tel = S.Telemetry(timing=True)
    times = []
    with ClockSampler(0) as clk:
        res = None
        for _ in range(args.steps):
            # drop the previous result first: while it is alive the caching allocator cannot reuse its
            # blocks and the call pays a cudaMalloc inside the timed region (seen as 0.5-70 ms on step 2)
            res = None
            res = one(tel, times)
    ms = sum(times) / len(times)
    groups = int(res.key_tensor.numel()) if res.key_tensor is not None else 0
    valid = None if args.no_validate else agg_validate(src, res, c["kind"])
    value = n / (ms / 1e3) / 1e9
    peak_gbs, peak_kind = measured_peaks()
    dist_ms = tel.phase_ms.get("distribute", 0.0) / args.steps
    rec_b = c["key_bits"] // 8 + (8 if c["values"] != "none" else 0)
    # records through the light distribute (folded nodes are read once by k_fold_nodes instead)
    moved = (tel.bucket_assignments - tel.fold_records) / args.steps
    achieved = (moved * 2 * rec_b) / (dist_ms / 1e3) / 1e9 if dist_ms > 0 else None
    fold_ms = tel.phase_ms.get("leaves", 0.0) / args.steps
    folded = tel.fold_records / args.steps
    fold_gbs = folded * rec_b / (fold_ms / 1e3) / 1e9 if fold_ms > 0 and folded else None
    e2e = None
    if not args.no_e2e:
        hk = torch.empty(n, dtype=src.keys.dtype, pin_memory=True)
        hk.copy_(src.keys)
        hv = None
        if src.values is not None:
            hv = torch.empty(n, dtype=src.values.dtype, pin_memory=True)
            hv.copy_(src.values)
        ts = []
        for i in range(3):
            with env.timed(ts if i else []):
                data = S.RecordArray(hk, hv)
                r = S.collect_reduce(data, adp, spec, params)
                ok = r.key_tensor.to("cpu", non_blocking=True)
                oa = r.agg_tensor.to("cpu", non_blocking=True)
            del data, r, ok, oa
        e_ms = sum(ts) / len(ts)
        in_b = n * rec_b
        out_b = groups * (c["key_bits"] // 8 + 8)
        e2e = {"value": n / (e_ms / 1e3) / 1e9, "unit": "Grecords/s", "h2d_bytes_per_step": in_b,
               "d2h_bytes_per_step": out_b, "ms_per_step": e_ms,
               "path": "RecordArray(pinned host tensors) -> collect_reduce -> (keys, aggs) to host"}
    cpu = None if args.no_cpu else agg_cpu_baseline(w, 1 << 22)
    line = {"metric": c["metric"], "value": value, "unit": "Grecords/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "ms_steps": [round(t, 3) for t in times],
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64" if c["key_bits"] == 64 else "u32",
            "data": "synthetic (device-generated, seeded)",
            "config": {"workload": c["desc"], "n_per_gpu": n, "groups": groups,
                       "params": "TuningParams.for_input(n) (reference defaults, seed 1)",
                       "l2": "256 MB buffer written before each step (flushes the 126 MB L2); input >= 4 GB"},
            "roofline": {"bound": "hbm", "kernel": "k_distribute1 (light-only scatter, all levels)",
                         "achieved": achieved, "peak": peak_gbs, "unit": "GB/s",
                         "frac": (achieved / peak_gbs) if achieved else None,
                         "traffic": (_traffic(w) or (None,))[0] if n == N_DEFAULT else None,
                         "alg_bytes_per_launch": moved * 2 * rec_b,
                         "peak_kind": peak_kind,
                         "bytes_model": f"{2 * rec_b} B per bucketed record (read + write {rec_b} B)"},
            "step_roofline": {"bytes_per_record": c["b_alg"], "achieved_gbs": c["b_alg"] * n / (ms / 1e3) / 1e9,
                              "peak": peak_gbs, "frac_of_measured": c["b_alg"] * n / (ms / 1e3) / 1e9 / peak_gbs,
                              "frac_of_nominal_8tbs": c["b_alg"] * n / (ms / 1e3) / NOMINAL_HBM},
            "fold_roofline": {"kernel": "k_fold_nodes (+ pair emission; the 'leaves' phase)", "records": folded,
                              "achieved": fold_gbs, "peak": peak_gbs, "unit": "GB/s",
                              "frac": (fold_gbs / peak_gbs) if fold_gbs else None,
                              "bytes_model": f"{rec_b} B per folded record (one read)"},
            "phase_ms_per_step": {k: v / args.steps for k, v in tel.phase_ms.items()},
            "gpu_launches": tel.kernel_launches, "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu,
            "validated": valid,
            "validation": "independent device reduction (torch bincount / sort + segmented sum), per-key equal"}
    print(json.dumps(line), flush=True)


def graph_main(args):
    """--workload graph: CSR transpose on a synthetic graph.

    The paper's graphs (LJ/TW/CM/SD) are not in this container; a seeded
    graph with Zipf(1.2) out-degrees and uniform targets over n/16 vertices
    stands in (power-law sources, the social-graph shape).  Unit: Gedges/s
    of transpose, input CSR resident, output allocated by the call.
    """
    import numpy as np
    import torch

    import paper_2304_10078_b200 as S
    from paper_2304_10078_b200.datagen import generate_device
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    env = Env(0, 1, dev, False)
    m = args.n
    nv = max(1, m // 16)
    src = generate_device("zipfian", 1.2, m, key_bits=32, seed=1, universe=nv, values="none", device=dev).keys
    src = (src.to(torch.int64) - 1).to(torch.uint32)            # ranks 1..nv -> ids 0..nv-1
    dst = generate_device("uniform", float(nv), m, key_bits=32, seed=2, values="none", device=dev).keys
    g = S.from_edges(nv, src, dst)
    del src, dst
    params = S.TuningParams.for_input(m)

    def one(tel=None, times=None):
        env.sync()
        with env.timed(times if times is not None else []):
            t = S.transpose(g, params, telemetry=tel)
        return t

    for _ in range(args.warmup):   # same code path as the timed steps (phase events on)
        one(S.Telemetry(timing=True))
    tel = S.Telemetry(timing=True)
    times = []
    with ClockSampler(0) as clk:
        for _ in range(args.steps):
            t = one(tel, times)
            del t
    ms = sum(times) / len(times)
    cpu = None
    if not args.no_cpu:   # the oracle transpose on a bounded sample (same shape, seed 1)
        import oracle as O
        ms_n = 1 << 20
        rng = np.random.default_rng(1)
        s_src = np.minimum(rng.zipf(1.2, ms_n) - 1, ms_n // 16 - 1).astype(np.uint32)
        s_dst = rng.integers(0, ms_n // 16, ms_n).astype(np.uint32)
        off, tg = O.csr_from_edges(ms_n // 16, s_src, s_dst)
        t0 = time.perf_counter()
        O.graph_transpose(ms_n // 16, off, tg)
        tc = time.perf_counter() - t0
        cpu = {"value": ms_n / tc / 1e9, "unit": "Gedges/s", "cores": 1, "kind": "port",
               "sample": f"transpose of a {ms_n}-edge graph of the same shape; reference algorithm restated "
                         f"in numpy (oracle/graphs_oracle.py), single thread, {tc:.2f} s"}
    line = {"metric": "graph transpose Gedges/s (m=1e9 u32 edges, Zipf out-degrees)", "value": m / (ms / 1e3) / 1e9,
            "unit": "Gedges/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (device-generated, seeded)",
            "config": {"workload": f"graph: transpose, m={m} edges, n={nv} vertices, out-degree Zipf(1.2), "
                                   "uniform targets", "params": "TuningParams.for_input(m)",
                       "l2": "input (>= 4 GB) larger than the 126 MB L2"},
            "phase_ms_per_step": {k: v / args.steps for k, v in tel.phase_ms.items()},
            "gpu_launches": tel.kernel_launches, "clocks": clk.summary(), "e2e": None, "cpu_baseline": cpu}
    print(json.dumps(line), flush=True)


def c1_main(args):
    """--workload c1: BASELINE.json configs[0], the reference's CPU-runnable
    case -- semisort of 2^20 (u64 key uniform in [0, 2^20), u64 value =
    index), default TuningParams (seed 1).  Launch-bound on a GPU (~75 MB
    of traffic; one host round trip per recursion level), so the line
    reports the per-call latency next to the reference package timed on
    the same input (all host cores), and whether the GPU output bytes equal
    the reference's (`validated`)."""
    import numpy as np
    import torch

    import paper_2304_10078_b200 as S
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    env = Env(0, 1, dev, False)
    n = 1 << 20
    rng = np.random.default_rng(1)
    keys = rng.integers(0, n, n).astype(np.uint64)
    vals = np.arange(n, dtype=np.uint64)
    pristine = S.RecordArray(keys, vals)
    work = pristine.copy()
    params = S.TuningParams.for_input(n)
    adp = S.UIntKeyAdapter()

    def one(tel=None, times=None):
        work.keys.copy_(pristine.keys)
        work.values.copy_(pristine.values)
        env.sync()
        with env.timed(times if times is not None else []):
            S.semisort(work, adp, "eq", params, telemetry=tel)

    for _ in range(max(args.warmup, 3)):
        one()
    tel = S.Telemetry(timing=True)
    times = []
    steps = max(args.steps, 20)
    with ClockSampler(0) as clk:
        for _ in range(steps):
            one(tel, times)
    ms = statistics.median(times)
    out_k, out_v = work.keys_host(), work.values_host()
    # e2e: pinned host input -> public API -> host output, per call
    hk, hv = torch.from_numpy(keys).pin_memory(), torch.from_numpy(vals).pin_memory()
    ok_k, ok_v = torch.empty_like(hk).pin_memory(), torch.empty_like(hv).pin_memory()
    e_times = []
    for i in range(steps + 3):
        env.sync()
        t0 = time.perf_counter()
        d = S.RecordArray(hk.to(dev, non_blocking=True), hv.to(dev, non_blocking=True))
        S.semisort(d, adp, "eq", params)
        ok_k.copy_(d.keys, non_blocking=True)
        ok_v.copy_(d.values, non_blocking=True)
        env.sync()
        if i >= 3:
            e_times.append((time.perf_counter() - t0) * 1e3)
    e_ms = statistics.median(e_times)
    cpu, validated = None, None
    R = _reference_module()
    if R is not None and not args.no_cpu:
        workers = os.cpu_count() or 1
        rt = []
        for i in range(4):   # the reference protocol: 4 reps, median of the last 3 (cli.py:79-80)
            data = R.RecordArray(keys.copy(), vals.copy())
            t0 = time.perf_counter()
            R.semisort(data, R.UIntKeyAdapter(), "eq", R.TuningParams.for_input(n, seed=1), workers=workers)
            rt.append(time.perf_counter() - t0)
        tc = statistics.median(rt[1:])
        validated = bool(np.array_equal(np.asarray(data.keys), out_k) and np.array_equal(np.asarray(data.values),
                                                                                         out_v))
        cpu = {"value": n / tc / 1e9, "unit": "Grecords/s", "cores": workers, "kind": "reference",
               "sample": f"the full c1 input: reference package semisort (baseline/_ref, workers={workers}), "
                         f"median of the last 3 of 4 reps ({tc:.3f} s); host {_cpu_model()}"}
    line = {"metric": "semisort Grecords/s (n=2^20 u64 k/v, uniform [0,2^20))", "value": n / (ms / 1e3) / 1e9,
            "unit": "Grecords/s", "n_gpus": 1, "steps": steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (numpy default_rng(1), uniform keys, value = index)",
            "config": {"workload": "c1: semisort n=2^20, uint64 key uniform [0, 2^20), value = index "
                                   "(BASELINE.json configs[0]); median call latency",
                       "params": "TuningParams.for_input(n) (seed 1)",
                       "l2": "16 MB input, L2-resident: a launch-latency-bound config, not a roofline one"},
            "phase_ms_per_step": {k: v / steps for k, v in tel.phase_ms.items()},
            "gpu_launches": tel.kernel_launches // steps if tel.kernel_launches else None,
            "clocks": clk.summary(),
            "e2e": {"value": n / (e_ms / 1e3) / 1e9, "unit": "Grecords/s", "h2d_bytes_per_step": 16 * n,
                    "d2h_bytes_per_step": 16 * n, "ms_per_step": e_ms},
            "cpu_baseline": cpu, "validated": validated,
            "validation": "GPU output bytes == the reference package's output bytes (same input, same params)"}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# launcher
# ---------------------------------------------------------------------------

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(args_list, gpus):
    """`bench.py --gpus N` without WORLD_SIZE: one process per GPU under
    torch.distributed.run (NCCL rendezvous on 127.0.0.1); rank 0 prints."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *args_list]
    return subprocess.call(cmd)


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N_DEFAULT, help="records per GPU (weak scaling)")
    ap.add_argument("--total", type=int, default=C5_TOTAL, help="records in total (strong scaling)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--e2e-n", type=int, default=None, help="records per GPU for the e2e leg (default n)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-n", type=int, default=1 << 24)
    ap.add_argument("--ref-n", type=int, default=None, help="records per --impl reference step (default: sized "
                                                            "so the run takes ~2-3 min)")
    ap.add_argument("--no-validate", action="store_true", help="skip the O(n) check of the last output")
    ap.add_argument("--validate", action="store_true", help="(default; kept for compatibility)")
    ap.add_argument("--mode", default="eq", choices=["eq", "lt"],
                    help="semisort mode: eq (default, the headline) or lt (semisort<, stable sort inside leaves)")
    ap.add_argument("--workload", default="c2", choices=["c2", "c5", "c3", "c4", "c1", "graph"],
                    help="c2 (default, the headline semisort); c5 multi-GPU mix; c3 collect_reduce sum64; "
                         "c4 histogram; c1 the 2^20 CPU-runnable case; graph: CSR transpose")
    return ap.parse_args(argv)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse_args(argv)
    if args.impl == "reference":
        reference_arm(args)
        return 0
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(argv, args.gpus)
    if args.workload in ("c3", "c4", "c1", "graph"):
        if int(os.environ.get("RANK", "0")) == 0:
            {"graph": graph_main, "c1": c1_main}.get(args.workload, agg_main)(args)
        return 0
    env = cuda_env()
    try:
        run_semisort(args, env, DeviceHooks(env), emit=lambda s: print(s, flush=True))
    finally:
        if env.dist_on:
            import torch.distributed as dist
            dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
