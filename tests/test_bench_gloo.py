"""bench.py's multi-rank orchestration over gloo (world_size 2, CPU).

The device pieces are replaced by CPU stand-ins (generator = a pure
function of the global index, the packed partition and the packed semisort
by numpy and the oracle, the shard validator by numpy); everything else is
bench.py's own code: shard sizes and first indices, the restore / barrier /
timed step loop, max over ranks, the ONE packed all_to_all_v exchange
(paper_2304_10078_b200.distributed), the per-rank checks plus the global
fingerprint comparison, and the JSON line rank 0 emits."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O

M64 = (1 << 64) - 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def gen_key(g: np.ndarray) -> np.ndarray:
    """c5-like: half uniform 64-bit, half a small skewed universe."""
    h = O.mix64_np(g.astype(np.uint64))
    sel = O.mix64_np(g.astype(np.uint64) ^ np.uint64(0x5EED)) & np.uint64(1)
    small = (h % np.uint64(97)) * (h % np.uint64(3))
    return np.where(sel == 1, h, small).astype(np.uint64)


class CpuHooks:
    """bench.DeviceHooks' interface on CPU tensors."""

    def __init__(self, env):
        import paper_2304_10078_b200 as S
        self.S = S
        self.env = env

    def generate(self, w, n, first, out=None):
        from paper_2304_10078_b200.core import _raw
        g = np.arange(first, first + n, dtype=np.uint64)
        k = torch.from_numpy(gen_key(g))
        v = torch.from_numpy(g.copy())
        if out is None:
            return _raw(k, v, "u64")
        out.keys.copy_(k)
        out.values.copy_(v)
        return out

    def restore(self, src, work):
        work.keys.copy_(src.keys)
        work.values.copy_(src.values)

    def telemetry(self):
        return self.S.Telemetry(timing=True)

    def dist_sort(self, work, mode, tel, recv_block=None, scratch=None):
        from paper_2304_10078_b200.distributed import dist_semisort
        from test_distributed_gloo import cpu_pack, cpu_sort_packed
        return dist_semisort(work, recv_block=recv_block, scratch=scratch, pack=cpu_pack, sort_packed=cpu_sort_packed)

    def shard_check(self, w, out, parts, rank):
        k = out.keys.numpy()
        v = out.values.numpy()
        bad_rec = int(np.sum(gen_key(v) != k))
        brk = np.ones(len(k), dtype=bool)
        brk[1:] = k[1:] != k[:-1]
        runs = int(brk.sum())
        bad_st = int(np.sum((~brk[1:]) & (v[1:] <= v[:-1]))) if len(k) > 1 else 0
        bits = parts.bit_length() - 1
        bad_dest = int(np.sum((O.mix64_np(k) >> np.uint64(64 - bits)) != rank)) if bits else 0
        s1 = int(v.astype(object).sum()) & M64
        s2 = int((v.astype(object) ** 2).sum()) & M64
        s3 = int(O.mix64_np(v).astype(object).sum()) & M64
        return [bad_rec, runs, bad_st, bad_dest, s1, s2, s3, len(np.unique(k))]

    def index_fingerprint(self, lo, hi):
        v = np.arange(lo, hi, dtype=np.uint64)
        return [int(v.astype(object).sum()) & M64, int((v.astype(object) ** 2).sum()) & M64,
                int(O.mix64_np(v).astype(object).sum()) & M64]


def _worker(rank, world, port, q, scaling):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        env = bench.Env(rank, world, torch.device("cpu"), True)
        args = bench.parse_args(["--gpus", str(world), "--steps", "2", "--warmup", "1", "--workload", "c5",
                                 "--n", "3000", "--total", "6000", "--scaling", scaling, "--no-e2e", "--no-cpu"])
        lines = []
        bench.run_semisort(args, env, CpuHooks(env), emit=lines.append)
        if rank == 0:
            q.put(lines)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_bench_orchestration_gloo_two_ranks(scaling):
    import json
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, scaling)) for r in range(2)]
    for p in procs:
        p.start()
    lines = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["steps"] == 2 and line["warmup"] == 1
    assert line["scaling"] == scaling
    assert line["validated"] is True, line["validation"]
    assert line["validation"]["fingerprints_match"] is True
    total = 6000 if scaling == "strong" else 2 * 3000
    assert line["config"]["n_total"] == total
    assert line["value"] == pytest.approx(total / (line["ms_per_step"] / 1e3) / 1e9)
    assert line["step_roofline"]["bytes_per_record_nvlink"] == 8.0    # 16 (G-1)/G at G = 2
    assert line["step_roofline"]["bytes_per_record_hbm"] == 72 + 40 + 16


def test_bench_single_process_args_and_relaunch_command(monkeypatch):
    """--gpus N without WORLD_SIZE re-launches under torch.distributed.run."""
    import bench
    calls = []
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    assert bench.main(["--gpus", "4", "--steps", "2"]) == 0
    cmd = calls[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-3:] == ["--gpus", "4", "--steps", "2"][-3:]
