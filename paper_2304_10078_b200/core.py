"""Drop-in semisort surface (the reference's core.py), executed on the GPU.

Every function keeps the reference signature and error behaviour
(core.py:139-598) and calls one C-ABI entry of libsemisort_b200.so; there
is no CPU execution path.  ``workers`` is accepted and ignored (the CUDA
grid replaces the thread pool; output is independent of it, as in the
reference).  For a fixed seed the output is byte-identical to the
reference's: sampling replays numpy's Philox stream on the device, and
bucket ids, counts, scans, distribution and the chained-hash base case
follow the reference definitions exactly.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .adapters import BytesKeyAdapter, KeyAdapter, UInt128KeyAdapter, UIntKeyAdapter, device_identity_flag
from .errors import ConfigurationError, ContractError
from .params import TuningParams
from .records import RecordArray, as_device_column, signed_view

DEPTH_LIMIT = 64   # core.py:39
U64_MASK = (1 << 64) - 1


def _mix64(x: int) -> int:
    from .adapters import _mix64 as m
    return m(x)


def mix64_pair(a: int, b: int) -> int:
    return _mix64((a ^ _mix64(b)) & U64_MASK)


@dataclass
class Telemetry:
    """Counters with the reference's semantics (core.py:42-61); repeated calls
    with the same object accumulate, exactly like the reference.  The extra
    fields are GPU-side diagnostics."""

    max_depth: int = 0
    nodes: int = 0
    scratch_allocations: int = 0
    scratch_moves: int = 0
    bucket_assignments: int = 0
    matrix_cells_by_level: dict = field(default_factory=dict)
    # GPU diagnostics
    kernel_launches: int = 0
    levels: int = 0
    leaves_smem: int = 0
    leaves_global: int = 0
    nodes_folded: int = 0
    fold_records: int = 0
    timing: bool = False
    phase_ms: dict = field(default_factory=dict)

    def observe_level(self, level: int, count: int = 1) -> None:
        self.nodes += count
        if level > self.max_depth:
            self.max_depth = level

    def add_matrix_cells(self, level: int, cells: int) -> None:
        self.matrix_cells_by_level[level] = self.matrix_cells_by_level.get(level, 0) + cells

    def _c(self):
        t = _lib.SSTelemetry()
        t.timing = 1 if self.timing else 0
        return t

    def _absorb(self, t) -> None:
        self.max_depth = max(self.max_depth, int(t.max_depth))
        self.nodes += int(t.nodes)
        self.scratch_allocations += int(t.scratch_allocations)
        self.scratch_moves += int(t.scratch_moves)
        self.bucket_assignments += int(t.bucket_assignments)
        for lvl in range(1, 65):
            c = int(t.matrix_cells_by_level[lvl])
            if c:
                self.add_matrix_cells(lvl, c)
        self.kernel_launches += int(t.kernel_launches)
        self.levels += int(t.levels)
        self.leaves_smem += int(t.leaves_smem)
        self.leaves_global += int(t.leaves_global)
        self.nodes_folded += int(t.nodes_folded)
        self.fold_records += int(t.fold_records)
        if self.timing:
            for i, name in enumerate(_lib.PHASES):
                self.phase_ms[name] = self.phase_ms.get(name, 0.0) + float(t.phase_ms[i])


class HeavyTable:
    """Heavy keys -> ids n_light .. n_light + n_heavy in discovery order
    (core.py:64-104).  ``keys`` is a host list; ``device_keys()`` the column
    the kernels read."""

    def __init__(self, n_light: int):
        self.n_light = n_light
        self._ids: dict = {}
        self.keys: list = []
        self.hashes: list = []
        self._dev = None

    def __len__(self) -> int:
        return len(self.keys)

    def insert(self, key, key_hash: int) -> int:
        bucket = self.n_light + len(self.keys)
        self._ids[int(key)] = bucket
        self.keys.append(int(key))
        self.hashes.append(int(key_hash))
        self._dev = None
        return bucket

    def lookup(self, key):
        return self._ids.get(int(key))

    def finalize(self, adapter=None) -> "HeavyTable":
        self._dev = None
        return self

    def device_keys(self, device) -> torch.Tensor:
        if self._dev is None or self._dev.device != device:
            arr = np.asarray(self.keys if self.keys else [0], dtype=np.uint64)
            self._dev = torch.from_numpy(arr).to(device)
        return self._dev


@dataclass
class BucketPlan:
    heavy: HeavyTable
    counts: object
    prefix: object
    offsets: object


@dataclass
class WorkBuffers:
    primary: RecordArray
    scratch: RecordArray
    live_in_primary: bool = True

    @property
    def live(self) -> RecordArray:
        return self.primary if self.live_in_primary else self.scratch

    @property
    def spare(self) -> RecordArray:
        return self.scratch if self.live_in_primary else self.primary


# ---------------------------------------------------------------------------
# plumbing
# ---------------------------------------------------------------------------

def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _layout(data: RecordArray, allow_u128: bool = False) -> tuple[int, int]:
    if not isinstance(data, RecordArray):
        raise ContractError("data must be a paper_2304_10078_b200.RecordArray")
    if data.key_kind not in (("u32", "u64", "u128") if allow_u128 else ("u32", "u64")):
        raise ContractError(f"{data.key_kind} keys are not supported by the GPU path")
    vb = data.value_bytes
    if vb not in (0, 4, 8, 16):
        raise ContractError(f"value rows of {vb} bytes are not supported by the GPU path")
    return data.key_bytes, vb


def _check_params(params: TuningParams | None, n: int) -> TuningParams:
    if params is None:
        return TuningParams.for_input(n)
    if params.input_size != n:
        raise ConfigurationError(f"params derived for n={params.input_size} used on n={n}")
    return params


def _philox_key(rng) -> int:
    """Key of a fresh numpy Philox Generator (the sample stream, core.py:238)."""
    bg = getattr(rng, "bit_generator", None)
    if not isinstance(bg, np.random.Philox):
        raise ContractError("the GPU sampler replays numpy's Philox streams only")
    st = bg.state
    if int(np.asarray(st["state"]["counter"]).any()) or st["buffer_pos"] != 4 or st["has_uint32"]:
        raise ContractError("the GPU sampler needs a freshly constructed Philox generator")
    key = np.asarray(st["state"]["key"], dtype=np.uint64)
    if int(key[1]):
        raise ContractError("Philox keys wider than 64 bits are not supported")
    return int(key[0])


def _heavy_args(heavy: HeavyTable | None, device):
    if heavy is None or len(heavy) == 0:
        return None, 0
    if len(heavy) > 512:
        raise ConfigurationError("more than 512 heavy keys")
    return heavy.device_keys(device), len(heavy)


# ---------------------------------------------------------------------------
# phase-level API (core.py:139-429)
# ---------------------------------------------------------------------------

def sample_and_bucket(data: RecordArray, adapter: KeyAdapter, params: TuningParams,
                      depth: int = 0, rng: np.random.Generator | None = None) -> HeavyTable:
    """core.py:221-260 on the device: heavy keys in discovery order."""
    device_identity_flag(adapter)
    kb, _ = _layout(data)
    n = len(data)
    key = params.seed & U64_MASK if rng is None else _philox_key(rng)
    table = HeavyTable(params.light_buckets)
    if n == 0 or params.max_heavy == 0 or min(n, params.sample_count) == 0:
        return table.finalize(adapter)
    if params.max_heavy > 512:
        raise ConfigurationError("max_heavy > 512 exceeds the shared-memory heavy table")
    dev = data.device
    out = torch.empty(max(params.max_heavy, 1), dtype=torch.uint64, device=dev)
    cnt = C.c_uint32(0)
    pc = params.as_c()
    wsb = _lib.lib().ss_phase_workspace_bytes(n, kb, 0, C.byref(pc))
    ws = _workspace(wsb, dev)
    _lib.check(_lib.lib().ss_sample_heavy(data.keys.data_ptr(), n, kb, C.byref(pc), key, out.data_ptr(),
                                          C.byref(cnt), ws.data_ptr(), ws.numel(), _stream(dev)))
    for k in out[: cnt.value].cpu().numpy().tolist():
        table.insert(k, adapter.hash_scalar(k))
    return table.finalize(adapter)


def assign_bucket_ids(data: RecordArray, heavy: HeavyTable, adapter: KeyAdapter, params: TuningParams,
                      depth: int = 0, pool=None) -> torch.Tensor:
    """core.py:169-190: int32 bucket id per record (device tensor)."""
    ident = device_identity_flag(adapter)
    kb, _ = _layout(data)
    n = len(data)
    dev = data.device
    ids = torch.empty(n, dtype=torch.int32, device=dev)
    if n == 0:
        return ids
    hk, nh = _heavy_args(heavy, dev)
    pc = params.as_c()
    _lib.check(_lib.lib().ss_assign_bucket_ids(data.keys.data_ptr(), n, kb, ident, C.byref(pc), depth,
                                               _ptr(hk), nh, ids.data_ptr(), None, 0, _stream(dev)))
    return ids


def get_bucket_id(key, heavy: HeavyTable | None, adapter: KeyAdapter, params: TuningParams,
                  depth: int = 0) -> int:
    """core.py:154-166 for one canonical key (a one-element device launch)."""
    ident = device_identity_flag(adapter)
    dev = torch.device("cuda", torch.cuda.current_device())
    k = torch.tensor([int(key) & U64_MASK], dtype=torch.uint64, device=dev)
    ids = torch.empty(1, dtype=torch.int32, device=dev)
    hk, nh = _heavy_args(heavy, dev)
    pc = params.as_c()
    _lib.check(_lib.lib().ss_assign_bucket_ids(k.data_ptr(), 1, 8, ident, C.byref(pc), depth, _ptr(hk), nh,
                                               ids.data_ptr(), None, 0, _stream(dev)))
    return int(ids.item())


def _check_ids(ids: torch.Tensor, n_buckets: int) -> None:
    """Bucket ids must lie in [0, n_buckets): the kernels index shared-memory
    counters by them (the reference rejects such ids in bincount / indexing)."""
    if ids.numel() == 0:
        return
    lo, hi = torch.aminmax(ids)
    lo, hi = int(lo.item()), int(hi.item())
    if lo < 0 or hi >= n_buckets:
        raise ConfigurationError(f"bucket ids must lie in [0, {n_buckets}); got [{lo}, {hi}]")


def _counts(data: RecordArray, ids, params: TuningParams, n_buckets: int, heavy, adapter, depth):
    n = len(data) if data is not None else len(ids)
    dev = data.device if data is not None else ids.device
    rows = params.num_subarrays(n)
    counts = torch.zeros((rows, n_buckets), dtype=torch.int64, device=dev)
    if n == 0:
        return counts
    # ids-only counting reads the 4-byte id column as u32 "keys"
    kb = data.key_bytes if data is not None else 4
    if ids is not None:
        _check_ids(ids, n_buckets)
    hk, nh = _heavy_args(heavy, dev)
    ident = device_identity_flag(adapter) if adapter is not None else 0
    pc = params.as_c()
    wsb = _lib.lib().ss_phase_workspace_bytes(n, kb, 0, C.byref(pc))
    wsb += (rows + 2) * (max(n_buckets, 1) + 2) * 24 + (1 << 20)
    ws = _workspace(wsb, dev)
    keys_ptr = data.keys.data_ptr() if data is not None else ids.data_ptr()
    _lib.check(_lib.lib().ss_count_matrix(keys_ptr, _ptr(ids), n, kb, ident, C.byref(pc), depth, _ptr(hk), nh,
                                          n_buckets, counts.data_ptr(), ws.data_ptr(), ws.numel(), _stream(dev)))
    return counts


def count_into_matrix(data: RecordArray, heavy: HeavyTable, adapter: KeyAdapter, params: TuningParams,
                      depth: int = 0, pool=None) -> torch.Tensor:
    """core.py:294-299: exact (subarray x bucket) counts, int64 device tensor."""
    _layout(data)
    return _counts(data, None, params, params.light_buckets + len(heavy), heavy, adapter, depth)


def counts_from_ids(ids, params: TuningParams, n_buckets: int, pool=None) -> torch.Tensor:
    """core.py:268-291 (_counts_from_ids) on device ids."""
    ids = as_device_column(np.asarray(ids, dtype=np.int32).view(np.uint32)).view(torch.int32) \
        if not isinstance(ids, torch.Tensor) else ids.to(torch.int32).contiguous()
    return _counts(None, ids, params, n_buckets, None, None, 0)


_counts_from_ids = counts_from_ids


def column_major_exclusive_scan(counts):
    """core.py:302-318: (prefix, offsets) as int64 device tensors."""
    if isinstance(counts, torch.Tensor):
        c = counts.to(torch.int64).contiguous()
        if not c.is_cuda:
            c = c.cuda()
    else:
        c = torch.from_numpy(np.ascontiguousarray(np.asarray(counts, dtype=np.int64))).cuda()
    rows, nb = c.shape
    dev = c.device
    prefix = torch.zeros((rows, nb), dtype=torch.int64, device=dev)
    offsets = torch.zeros(nb + 1, dtype=torch.int64, device=dev)
    if nb == 0:
        return prefix, offsets
    wsb = (rows + 2) * (nb + 2) * 16 + (rows // 8 + 2) * (nb + 2) * 8 + 65536
    ws = _workspace(wsb, dev)
    _lib.check(_lib.lib().ss_column_scan(c.data_ptr(), rows, nb, prefix.data_ptr(), offsets.data_ptr(),
                                         ws.data_ptr(), ws.numel(), _stream(dev)))
    return prefix, offsets


def _distribute(src: RecordArray, dst: RecordArray, ids, prefix, params: TuningParams, n_buckets: int,
                heavy, adapter, depth):
    kb, vb = _layout(src)
    n = len(src)
    if n == 0:
        return
    dev = src.device
    p = prefix.to(torch.int64).contiguous() if isinstance(prefix, torch.Tensor) else \
        torch.from_numpy(np.ascontiguousarray(np.asarray(prefix, dtype=np.int64)))
    p = p.to(dev)
    if ids is not None:
        _check_ids(ids, n_buckets)
    hk, nh = _heavy_args(heavy, dev)
    ident = device_identity_flag(adapter) if adapter is not None else 0
    pc = params.as_c()
    wsb = _lib.lib().ss_phase_workspace_bytes(n, kb, vb, C.byref(pc)) + \
        (params.num_subarrays(n) + 2) * (max(n_buckets, 1) + 2) * 24 + (1 << 20)
    ws = _workspace(wsb, dev)
    _lib.check(_lib.lib().ss_distribute(src.keys.data_ptr(), _ptr(src.values), dst.keys.data_ptr(),
                                        _ptr(dst.values), _ptr(ids), n, kb, vb, ident, C.byref(pc), depth,
                                        _ptr(hk), nh, n_buckets, p.data_ptr(), ws.data_ptr(), ws.numel(),
                                        _stream(dev)))


def distribute(data: RecordArray, prefix, heavy: HeavyTable, adapter: KeyAdapter, params: TuningParams,
               depth: int, dest: RecordArray, *, ids=None, pool=None) -> None:
    """core.py:365-380: stable scatter of data into dest by bucket cursors."""
    if len(dest) != len(data):
        raise ConfigurationError("destination must match the subproblem size")
    device_identity_flag(adapter)
    if ids is not None:
        ids = ids.to(torch.int32).contiguous() if isinstance(ids, torch.Tensor) else \
            torch.from_numpy(np.asarray(ids, dtype=np.int32)).to(data.device)
    _distribute(data, dest, ids, prefix, params, params.light_buckets + len(heavy), heavy, adapter, depth)


def distribute_ids(src: RecordArray, dst: RecordArray, base: int, ids, prefix, params: TuningParams,
                   n_buckets: int, pool=None) -> None:
    """core.py:339-362 (_distribute_ids): move the node's records
    src[base:base+len(ids)] to dst[base + cursor] (the window is len(ids)
    records wide on both sides, as in the reference)."""
    ids = ids.to(torch.int32).contiguous() if isinstance(ids, torch.Tensor) else \
        torch.from_numpy(np.asarray(ids, dtype=np.int32)).to(src.device)
    m = int(ids.shape[0])
    base = int(base)
    if base < 0 or base + m > len(src) or base + m > len(dst):
        raise ConfigurationError(f"window [{base}, {base + m}) exceeds the source/destination arrays")
    rows = params.num_subarrays(m)
    pshape = tuple(prefix.shape) if hasattr(prefix, "shape") else np.asarray(prefix).shape
    if m and pshape != (rows, n_buckets):
        raise ConfigurationError(f"prefix has shape {pshape}, expected {(rows, n_buckets)}")
    src, dst = src.view(base, base + m), dst.view(base, base + m)
    _distribute(src, dst, ids, prefix, params, n_buckets, None, None, 0)


_distribute_ids = distribute_ids


def _base_case(data: RecordArray, adapter: KeyAdapter, mode: int) -> None:
    ident = device_identity_flag(adapter)
    kb, vb = _layout(data)
    n = len(data)
    if n < 2:
        return
    dev = data.device
    ws = _workspace(_lib.lib().ss_base_case_workspace_bytes(n, kb, vb), dev)
    _lib.check(_lib.lib().ss_base_case(data.keys.data_ptr(), _ptr(data.values), n, kb, vb, mode, ident,
                                       ws.data_ptr(), ws.numel(), _stream(dev)))


def base_case_eq(data: RecordArray, adapter: KeyAdapter) -> None:
    """core.py:404-422: chained-hash group order, stable, in place."""
    _base_case(data, adapter, _lib.SS_MODE_EQ)


def base_case_lt(data: RecordArray, adapter: KeyAdapter) -> None:
    """core.py:425-429: stable sort by key, in place."""
    if not adapter.has_lt:
        raise ContractError(f"{type(adapter).__name__} has no less-than test")
    _base_case(data, adapter, _lib.SS_MODE_LT)


# ---------------------------------------------------------------------------
# the whole path (core.py:533-598)
# ---------------------------------------------------------------------------

def semisort(data: RecordArray, adapter: KeyAdapter, mode: str = "eq", params: TuningParams | None = None,
             *, workers: int | None = None, telemetry: Telemetry | None = None) -> RecordArray:
    """Reorder ``data`` in place so equal keys are contiguous (core.py:566-598).

    Stable and deterministic; for a fixed ``params.seed`` the output bytes
    equal the reference's.  Allocates one scratch of the input's size (in a
    torch workspace) per call.
    """
    if mode not in ("eq", "lt"):
        raise ConfigurationError(f"mode must be 'eq' or 'lt', got {mode!r}")
    if mode == "lt" and not adapter.has_lt:
        raise ContractError("mode 'lt' requires an adapter with a less-than test")
    if getattr(data, "key_kind", None) == "bytes" or isinstance(adapter, BytesKeyAdapter):
        return _semisort_bytes(data, adapter, mode, params, telemetry)
    ident = device_identity_flag(adapter, allow_u128=True)
    kb, vb = _layout(data, allow_u128=True)
    if (data.key_kind == "u128") != (adapter.key_kind == "u128"):
        raise ContractError(f"{type(adapter).__name__} does not match {data.key_kind} keys")
    n = len(data)
    params = _check_params(params, n)
    tel = telemetry if telemetry is not None else Telemetry()
    dev = data.device
    pc = params.as_c()
    wsb = _lib.lib().ss_semisort_workspace_bytes(n, kb, vb, C.byref(pc))
    if wsb == 0:
        _lib.check(_lib.SS_ERR_CONFIG)
    ws = _workspace(wsb, dev)
    ct = tel._c()
    _lib.check(_lib.lib().ss_semisort(data.keys.data_ptr(), _ptr(data.values), n, kb, vb,
                                      _lib.SS_MODE_LT if mode == "lt" else _lib.SS_MODE_EQ, ident, C.byref(pc),
                                      ws.data_ptr(), ws.numel(), C.byref(ct), _stream(dev)))
    tel._absorb(ct)
    return data


def _semisort_bytes(data, adapter, mode, params, telemetry):
    """Byte-view keys (adapters.py:200-275): semisort of 128-bit identity keys
    (content hash, length | content rank) carrying the record index, then the
    caller's views and values are permuted in place (bytes_keys.py)."""
    from . import bytes_keys
    if not isinstance(adapter, BytesKeyAdapter) or getattr(data, "key_kind", None) != "bytes":
        raise ContractError(f"{type(adapter).__name__} does not match {getattr(data, 'key_kind', None)} keys")
    if type(adapter).hash_scalar is not BytesKeyAdapter.hash_scalar:
        raise ContractError(f"{type(adapter).__name__}.hash_scalar is custom Python; the GPU path only runs the "
                            "reference's content hash")
    if data.values is not None and data.value_bytes not in (4, 8, 16):
        raise ContractError(f"value rows of {data.value_bytes} bytes are not supported by the GPU path")
    n = len(data)
    params = _check_params(params, n)
    syn = bytes_keys.synthetic_keys(data, mode)
    idx = torch.arange(n, dtype=torch.int64, device=data.device).view(torch.uint64)
    tmp = RecordArray(syn, idx, "u128")
    semisort(tmp, UInt128KeyAdapter(identity=True), mode, params, telemetry=telemetry)
    perm = tmp.values.view(torch.int64)
    if mode == "eq":
        bytes_keys.check_grouped(data, tmp.keys, perm)
    data.keys.copy_(data.keys.view(torch.int64)[perm].view(torch.uint64))
    if data.values is not None:
        data.values.copy_(signed_view(data.values)[perm].view(data.values.dtype))
    return data


def local_refine(buffers: WorkBuffers, plan: BucketPlan, adapter: KeyAdapter, mode: str, params: TuningParams,
                 *, depth: int = 0, workers: int | None = None, telemetry: Telemetry | None = None) -> None:
    """core.py:533-563: refine the light buckets of a distributed node."""
    if mode not in ("eq", "lt"):
        raise ConfigurationError(f"mode must be 'eq' or 'lt', got {mode!r}")
    ident = device_identity_flag(adapter)
    data = buffers.primary
    kb, vb = _layout(data)
    n = len(data)
    tel = telemetry if telemetry is not None else Telemetry()
    offs = plan.offsets
    offs = offs.cpu().numpy() if isinstance(offs, torch.Tensor) else np.asarray(offs)
    offs = np.ascontiguousarray(offs.astype(np.int64))
    nb = len(offs) - 1
    dev = data.device
    pc = params.as_c()
    wsb = _lib.lib().ss_semisort_workspace_bytes(n, kb, vb, C.byref(pc))
    ws = _workspace(wsb, dev)
    ct = tel._c()
    _lib.check(_lib.lib().ss_local_refine(
        data.keys.data_ptr(), _ptr(data.values), buffers.scratch.keys.data_ptr(), _ptr(buffers.scratch.values), n,
        kb, vb, _lib.SS_MODE_LT if mode == "lt" else _lib.SS_MODE_EQ, ident, C.byref(pc),
        offs.ctypes.data_as(C.POINTER(C.c_int64)), nb, 1 if buffers.live_in_primary else 0, depth,
        ws.data_ptr(), ws.numel(), C.byref(ct), _stream(dev)))
    tel._absorb(ct)


def _raw(keys, values, kind) -> RecordArray:
    r = RecordArray.__new__(RecordArray)
    r.keys, r.values, r.arena, r.key_kind = keys, values, None, kind
    return r


def semisort_packed(pairs: torch.Tensor, n: int, adapter: KeyAdapter, mode: str = "eq",
                    params: TuningParams | None = None, *, scratch: torch.Tensor | None = None,
                    telemetry: Telemetry | None = None) -> RecordArray:
    """Semisort of ``n`` packed (key, value) records held in the first 2n
    words of ``pairs`` (uint32 or uint64; what a rank receives from the
    multi-GPU exchange).  Same result and errors as ``semisort`` on the
    unpacked columns (core.py:566-598); the result is left as SoA columns in
    the same memory and returned as a RecordArray of views: keys = words
    [0, n), values = words [n, 2n).  ``scratch`` (>= 2n words of the same
    dtype, e.g. the exchange's send buffer) replaces the internal scratch."""
    if mode not in ("eq", "lt"):
        raise ConfigurationError(f"mode must be 'eq' or 'lt', got {mode!r}")
    if mode == "lt" and not adapter.has_lt:
        raise ContractError("mode 'lt' requires an adapter with a less-than test")
    ident = device_identity_flag(adapter)
    flat = pairs.reshape(-1)
    if flat.dtype not in (torch.uint32, torch.uint64) or not flat.is_cuda or not flat.is_contiguous():
        raise ContractError("packed records must be a contiguous uint32/uint64 CUDA tensor")
    if flat.numel() < 2 * n:
        raise ConfigurationError(f"{flat.numel()} words hold fewer than {n} packed records")
    kb = flat.element_size()
    params = _check_params(params, n)
    tel = telemetry if telemetry is not None else Telemetry()
    dev = flat.device
    scr = None
    if scratch is not None:
        s = scratch.reshape(-1)
        if s.dtype != flat.dtype or s.numel() < 2 * n or not s.is_contiguous():
            raise ConfigurationError("scratch must hold 2n words of the records' dtype")
        scr = s
    pc = params.as_c()
    lib = _lib.lib()
    wsb = lib.ss_semisort_pairs_workspace_bytes(n, kb, C.byref(pc), 0 if scr is not None else 1)
    if wsb == 0:
        _lib.check(_lib.SS_ERR_CONFIG)
    ws = _workspace(wsb, dev)
    ct = tel._c()
    _lib.check(lib.ss_semisort_pairs(flat.data_ptr(), n, kb, _lib.SS_MODE_LT if mode == "lt" else _lib.SS_MODE_EQ,
                                     ident, C.byref(pc), _ptr(scr), ws.data_ptr(), ws.numel(), C.byref(ct),
                                     _stream(dev)))
    tel._absorb(ct)
    return _raw(flat[:n], flat[n:2 * n], "u64" if kb == 8 else "u32")
