"""hgrd-b200 — the race-check stage of arXiv 2604.02106 (HGRD) on B200.

Python face of ``libhgrd_gpu.so`` (C ABI: ``include/hgrd_gpu.h``).  The names
mirror the reference's oracle API (reference include/hgrd/oracle.hpp):

* :class:`ExecConfig`, :class:`SweepCaps`   — oracle.hpp:17-25, :59-66
* :meth:`GpuContext.run_concrete`            — ``hgrd::runConcrete``      (:57)
* :meth:`GpuContext.enumerate_verdict`       — ``hgrd::enumerateVerdict`` (:75)
* :func:`count_inputs`                       — ``hgrd::countInputs``      (:79)

Results are the reference's ``OracleResult`` / ``SweepRace`` fields as JSON
dicts (plus ``witnesses`` and ``stats``).  There is no CPU fallback: without
the built library or without an sm_100 device these calls raise.
"""
from __future__ import annotations

import ctypes
import json
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
# (HGRD_GPU_LIBRARY: development A/B runs against another build of the same tree)
LIBRARY_PATH = os.environ.get("HGRD_GPU_LIBRARY") or os.path.join(_HERE, "libhgrd_gpu.so")

# ---------------------------------------------------------------- ABI types
c_int32, c_int64, c_uint8, c_uint16, c_uint32, c_uint64 = (
    ctypes.c_int32, ctypes.c_int64, ctypes.c_uint8, ctypes.c_uint16,
    ctypes.c_uint32, ctypes.c_uint64)

LAUNCH_SEQUENTIAL = 1
LAUNCH_PAIRWISE = 2
LAUNCH_NO_WITNESS = 4
LAUNCH_GENERAL = 8
RACE_KINDS = ("INTER-BLOCK", "INTRA-BLOCK", "INTRA-WARP")


class Insn(ctypes.Structure):
    _fields_ = [("op", c_uint8), ("sub", c_uint8), ("a", c_uint16), ("b", c_uint16),
                ("c", c_uint16), ("pad", c_uint16), ("imm", c_int64)]


class Site(ctypes.Structure):
    _fields_ = [("loc", c_int32), ("param", c_int32), ("kind", c_uint8),
                ("atomic_op", c_uint8), ("scope", c_uint8), ("pad0", c_uint8),
                ("pad1", c_int32)]


class Launch(ctypes.Structure):
    _fields_ = [("code", ctypes.POINTER(Insn)), ("n_code", c_uint32), ("n_regs", c_uint32),
                ("reg_init", ctypes.POINTER(c_int64)), ("sites", ctypes.POINTER(Site)),
                ("n_sites", c_uint32), ("n_locs", c_uint32),
                ("param_handle", ctypes.POINTER(c_int32)), ("n_params", c_uint32),
                ("flags", c_uint32), ("grid", c_int64 * 3), ("block", c_int64 * 3),
                ("warp_size", c_int64), ("step_budget", c_int64)]


class Race(ctypes.Structure):
    _fields_ = [("loc_a", c_int32), ("loc_b", c_int32), ("kind", c_int32),
                ("site_x", c_int32), ("site_y", c_int32), ("handle", c_int32),
                ("index", c_int64), ("thread_x", c_int64), ("thread_y", c_int64),
                ("seq_x", c_int32), ("seq_y", c_int32)]


class Trap(ctypes.Structure):
    _fields_ = [("site", c_int32), ("kind", c_int32), ("thread", c_int64)]


class Result(ctypes.Structure):
    _fields_ = [("races", ctypes.POINTER(Race)), ("race_cap", c_uint32), ("n_races", c_uint32),
                ("traps", ctypes.POINTER(Trap)), ("trap_cap", c_uint32), ("n_traps", c_uint32),
                ("n_traps_total", c_uint64), ("steps", c_int64), ("instances", c_uint64),
                ("records", c_uint64), ("aborted", c_int32), ("abort_stmt", c_int32),
                ("mode", c_uint32), ("device_ms", ctypes.c_float)]


class Shard(ctypes.Structure):
    """hgrd_gpu_shard: a whole-block range of one launch (sharded check)."""
    _fields_ = [("block_begin", c_int64), ("block_end", c_int64),
                ("inter_lo", ctypes.c_void_p), ("inter_hi", ctypes.c_void_p),
                ("inter_n", ctypes.c_uint64)]


HGRD_GPU_ENOTSUP = -95


class NotShardable(RuntimeError):
    """The launch (or this shard) needs the ordered path: run it unsharded."""


class _CudaArray:
    """__cuda_array_interface__ view of a context-owned device table."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i4", "data": (ptr, False),
                                         "version": 3, "strides": None}


# ----------------------------------------------------------- configuration
@dataclass
class ExecConfig:
    """reference ExecConfig, include/hgrd/oracle.hpp:17-25"""
    gridCap: Sequence[int] = (2, 2, 1)
    blockCap: Sequence[int] = (4, 1, 1)
    warpSize: int = 32
    inputs: Sequence[int] = ()
    maxThreads: int = 64
    maxArrayElems: int = 1 << 20
    maxSteps: int = 1 << 20

    def to_json(self) -> str:
        d = {k: list(v) if isinstance(v, (list, tuple)) else v for k, v in self.__dict__.items()}
        return json.dumps(d)


@dataclass
class SweepCaps:
    """reference SweepCaps, include/hgrd/oracle.hpp:59-66"""
    gridCap: Sequence[int] = (2, 2, 1)
    blockCap: Sequence[int] = (4, 1, 1)
    inputSet: Sequence[int] = (0, 1, 2, 3, 127)
    warpSizes: Sequence[int] = (2, 4)
    maxThreads: int = 64
    maxConfigs: int = 100000

    def to_json(self) -> str:
        d = {k: list(v) if isinstance(v, (list, tuple)) else v for k, v in self.__dict__.items()}
        return json.dumps(d)


def _cfg_json(cfg) -> str:
    if cfg is None:
        return "{}"
    if isinstance(cfg, str):
        return cfg
    if isinstance(cfg, dict):
        return json.dumps(cfg)
    return cfg.to_json()


# ------------------------------------------------------------------ library
_lib = None


def load_library() -> ctypes.CDLL:
    """Load the in-tree libhgrd_gpu.so (fails loudly when it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIBRARY_PATH):
        raise ImportError(f"{LIBRARY_PATH} is missing: run __graft_entry__.build() "
                          "(python paper_2604_02106_b200/build.py)")
    lib = ctypes.CDLL(LIBRARY_PATH)
    P = ctypes.c_void_p
    lib.hgrd_gpu_create.argtypes = [ctypes.c_int, ctypes.POINTER(P)]
    lib.hgrd_gpu_destroy.argtypes = [P]
    lib.hgrd_gpu_last_error.argtypes = [P]
    lib.hgrd_gpu_last_error.restype = ctypes.c_char_p
    lib.hgrd_gpu_buffers_reset.argtypes = [P]
    lib.hgrd_gpu_buffer_alloc.argtypes = [P, c_int64, ctypes.POINTER(c_int32)]
    lib.hgrd_gpu_buffer_write.argtypes = [P, c_int32, c_int64, c_int64, P]
    lib.hgrd_gpu_buffer_write_async.argtypes = [P, c_int32, c_int64, c_int64, P]
    lib.hgrd_gpu_buffer_read.argtypes = [P, c_int32, c_int64, c_int64, P]
    lib.hgrd_gpu_check_launch.argtypes = [P, ctypes.POINTER(Launch), ctypes.POINTER(Result)]
    for fn in ("hgrd_gpu_run_concrete_json", "hgrd_gpu_enumerate_verdict_json"):
        getattr(lib, fn).argtypes = [P, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p,
                                     ctypes.POINTER(P)]
    lib.hgrd_gpu_enumerate_verdict_many_json.argtypes = [P, ctypes.c_char_p, ctypes.c_int,
                                                         ctypes.c_int, ctypes.POINTER(P)]
    lib.hgrd_gpu_lower_json.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p,
                                        ctypes.POINTER(P)]
    lib.hgrd_gpu_sweep_shard_json.argtypes = [P, ctypes.c_char_p, ctypes.c_char_p,
                                              ctypes.c_char_p, ctypes.c_int, ctypes.c_int,
                                              ctypes.POINTER(P)]
    lib.hgrd_gpu_count_inputs.argtypes = [ctypes.c_char_p, ctypes.c_char_p]
    lib.hgrd_gpu_block_private.argtypes = [P, ctypes.POINTER(ctypes.c_uint8)]
    lib.hgrd_gpu_stream_sites.argtypes = [P, ctypes.POINTER(ctypes.c_int64)]
    lib.hgrd_gpu_shard_check.argtypes = [P, P, P, P]
    lib.hgrd_gpu_shard_inter.argtypes = [P, P, P, ctypes.POINTER(ctypes.c_uint64),
                                         ctypes.POINTER(c_uint32), ctypes.c_uint64,
                                         ctypes.POINTER(ctypes.c_uint64)]
    lib.hgrd_gpu_shard_inter_scan.argtypes = [P, P, P, P, ctypes.c_uint64, ctypes.c_uint64,
                                              ctypes.POINTER(ctypes.c_uint64), c_uint32]
    lib.hgrd_gpu_shard_inter_records.argtypes = [P, P, P, ctypes.POINTER(ctypes.c_uint64),
                                                 c_uint32, ctypes.POINTER(ctypes.c_uint64),
                                                 ctypes.POINTER(c_uint32), ctypes.c_uint64,
                                                 ctypes.POINTER(ctypes.c_uint64)]
    lib.hgrd_gpu_stream.argtypes = [P]
    lib.hgrd_gpu_stream.restype = ctypes.c_void_p
    lib.hgrd_gpu_shard_detect.argtypes = [P, P, ctypes.POINTER(ctypes.c_uint64),
                                          ctypes.POINTER(c_uint32), ctypes.c_uint64, P]
    I3 = ctypes.c_int64 * 3
    lib.hgrd_gpu_jit_check.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, I3, I3,
                                       ctypes.c_int64, ctypes.POINTER(P)]
    lib.hgrd_gpu_free.argtypes = [P]
    lib.hgrd_gpu_set_profiling.argtypes = [P, ctypes.c_int]
    lib.hgrd_gpu_last_profile.argtypes = [P]
    lib.hgrd_gpu_last_profile.restype = ctypes.c_char_p
    lib.hgrd_gpu_set_fused.argtypes = [P, ctypes.c_int]
    lib.hgrd_gpu_set_jit.argtypes = [P, ctypes.c_int]
    lib.hgrd_gpu_jit_info.argtypes = [P]
    lib.hgrd_gpu_jit_info.restype = ctypes.c_char_p
    lib.hgrd_gpu_kernel_launches.argtypes = [P]
    lib.hgrd_gpu_kernel_launches.restype = ctypes.c_ulonglong
    lib.hgrd_gpu_transfer_bytes.argtypes = [P, ctypes.POINTER(ctypes.c_ulonglong),
                                            ctypes.POINTER(ctypes.c_ulonglong)]
    _lib = lib
    return lib


def _take_string(lib, p: ctypes.c_void_p) -> str:
    s = ctypes.string_at(p.value).decode() if p.value else ""
    lib.hgrd_gpu_free(p)
    return s


def count_inputs(source: str, file_name: str = "prog.mcu") -> int:
    """reference hgrd::countInputs (src/oracle.cpp:805-861)."""
    return load_library().hgrd_gpu_count_inputs(source.encode(), file_name.encode())


def lower(source: str, kernel: str, file_name: str = "prog.mcu") -> dict:
    """Lowered bytecode + access sites of one kernel (no GPU needed)."""
    lib = load_library()
    out = ctypes.c_void_p()
    rc = lib.hgrd_gpu_lower_json(source.encode(), file_name.encode(), kernel.encode(),
                                 ctypes.byref(out))
    d = json.loads(_take_string(lib, out))
    if rc != 0:
        raise ValueError(f"lowering failed: {d}")
    return d


def jit_check(source: str, kernel: str, grid=(1, 1, 1), block=(256, 1, 1),
              warp_size: int = 32, file_name: str = "prog.mcu") -> dict:
    """Compile the NVRTC-specialised kernels of one kernel for sm_100a
    without loading them (no GPU needed); raises on a compile error."""
    lib = load_library()
    I3 = ctypes.c_int64 * 3
    out = ctypes.c_void_p()
    rc = lib.hgrd_gpu_jit_check(source.encode(), file_name.encode(), kernel.encode(),
                                I3(*grid), I3(*block), warp_size, ctypes.byref(out))
    d = json.loads(_take_string(lib, out))
    if rc != 0:
        raise RuntimeError(f"jit_check failed ({rc}): {d}")
    return d


class LaunchSpec:
    """A fully parameterised launch (the C ABI's hgrd_gpu_launch) + keep-alives."""

    def __init__(self, lowered: dict, grid, block, warp_size: int,
                 scalars: Optional[Dict[str, int]] = None,
                 handles: Optional[Dict[str, int]] = None,
                 step_budget: int = 1 << 60, flags: Optional[int] = None):
        self.lowered = lowered
        code = lowered["code"]
        self._code = (Insn * len(code))(*[Insn(op, sub, a, b, c, 0, imm)
                                         for op, sub, a, b, c, imm in code])
        sites = lowered["sites"]
        self._sites = (Site * max(len(sites), 1))(*[
            Site(s["loc"], s["param"], s["kind"], s["atomicOp"], s["scope"], 0, 0)
            for s in sites])
        regs = [0] * max(lowered["nRegs"], 1)
        scalars = scalars or {}
        handles = handles or {}
        ph = []
        for p in lowered["params"]:
            if p["array"]:
                ph.append(handles.get(p["name"], -1))
            else:
                ph.append(-1)
                if p["reg"] >= 0:
                    regs[p["reg"]] = int(scalars.get(p["name"], 0))
        self._regs = (c_int64 * len(regs))(*regs)
        self._ph = (c_int32 * max(len(ph), 1))(*ph)
        if flags is None:
            flags = LAUNCH_PAIRWISE if lowered["hasLocks"] else 0
        self.launch = Launch(self._code, len(code), lowered["nRegs"], self._regs,
                             self._sites, len(sites), len(lowered["locs"]), self._ph, len(ph),
                             flags, (c_int64 * 3)(*grid), (c_int64 * 3)(*block), warp_size,
                             step_budget)

    def block_private(self):
        """Per site: True when its buffer is proven block-private (host
        affine analysis, affine.cpp); no GPU needed."""
        lib = load_library()
        n = self.launch.n_sites
        out = (ctypes.c_uint8 * max(n, 1))()
        rc = lib.hgrd_gpu_block_private(ctypes.byref(self.launch), out)
        if rc:
            raise RuntimeError(f"block_private failed ({rc})")
        return [bool(out[i]) for i in range(n)]

    def stream_sites(self):
        """Per site: c when its index is always the dense thread id + c
        (a streamed load, affine.cpp streamSites), else None; no GPU needed."""
        lib = load_library()
        n = self.launch.n_sites
        out = (ctypes.c_int64 * max(n, 1))()
        rc = lib.hgrd_gpu_stream_sites(ctypes.byref(self.launch), out)
        if rc:
            raise RuntimeError(f"stream_sites failed ({rc})")
        return [None if out[i] == -(1 << 63) else int(out[i]) for i in range(n)]

    @property
    def n_threads(self) -> int:
        g, b = self.launch.grid, self.launch.block
        return g[0] * g[1] * g[2] * b[0] * b[1] * b[2]

    def new_result(self, trap_cap: int = 256):
        n = max(len(self.lowered["locs"]), 1)
        races = (Race * (3 * n * n))()
        traps = (Trap * max(trap_cap, 1))()
        res = Result(races, 3 * n * n, 0, traps, trap_cap, 0, 0, 0, 0, 0, 0, -1, 0, 0.0)
        return res, races, traps

    def decode(self, res: Result) -> dict:
        """Races as reference-shaped dicts (kind, locA, locB, array, address) + witness."""
        locs = self.lowered["locs"]
        sites = self.lowered["sites"]
        races = []
        for i in range(res.n_races):
            r = res.races[i]
            races.append({"kind": RACE_KINDS[r.kind], "locA": list(locs[r.loc_a]),
                          "locB": list(locs[r.loc_b]), "array": sites[r.site_x]["array"],
                          "handle": r.handle, "address": r.index,
                          "threadA": r.thread_x, "seqA": r.seq_x,
                          "threadB": r.thread_y, "seqB": r.seq_y})
        races.sort(key=lambda d: (d["locA"], d["locB"], RACE_KINDS.index(d["kind"])))
        traps = [(res.traps[i].site, res.traps[i].kind, res.traps[i].thread)
                 for i in range(res.n_traps)]
        return {"races": races, "traps": traps, "steps": res.steps,
                "instances": res.instances, "records": res.records,
                "aborted": bool(res.aborted), "abortStmt": res.abort_stmt,
                "mode": res.mode, "deviceMs": res.device_ms}


class GpuContext:
    """One B200 context (hgrd_gpu_ctx): device buffers + race-check calls."""

    def __init__(self, device: int = 0):
        self._lib = load_library()
        self._ctx = ctypes.c_void_p()
        rc = self._lib.hgrd_gpu_create(device, ctypes.byref(self._ctx))
        if rc != 0:
            raise RuntimeError(f"hgrd_gpu_create(device={device}) failed with {rc}: "
                               "no usable sm_100 device (there is no CPU fallback)")

    def close(self):
        if self._ctx:
            self._lib.hgrd_gpu_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _err(self, what: str, rc: int):
        msg = self._lib.hgrd_gpu_last_error(self._ctx)
        raise RuntimeError(f"{what} failed ({rc}): {msg.decode() if msg else ''}")

    # -- reference-shaped API --
    def run_concrete(self, source: str, config=None, file_name: str = "prog.mcu") -> dict:
        out = ctypes.c_void_p()
        rc = self._lib.hgrd_gpu_run_concrete_json(self._ctx, source.encode(),
                                                  file_name.encode(),
                                                  _cfg_json(config).encode(),
                                                  ctypes.byref(out))
        s = _take_string(self._lib, out)
        if rc != 0:
            raise RuntimeError(f"run_concrete failed ({rc}): {s}")
        return json.loads(s)

    def sweep_shard(self, source: str, caps=None, file_name: str = "prog.mcu",
                    rank: int = 0, world: int = 1) -> dict:
        """This rank's share of the enumerateVerdict lattice (see parallel.py)."""
        out = ctypes.c_void_p()
        rc = self._lib.hgrd_gpu_sweep_shard_json(self._ctx, source.encode(), file_name.encode(),
                                                 _cfg_json(caps).encode(), rank, world,
                                                 ctypes.byref(out))
        s = _take_string(self._lib, out)
        if rc != 0:
            raise RuntimeError(f"sweep_shard failed ({rc}): {s}")
        return json.loads(s)

    @staticmethod
    def sweep_jobs_payload(jobs) -> bytes:
        """The C ABI's jobs JSON for enumerate_verdict_many_raw."""
        return json.dumps([{"source": j["source"], "file": j.get("file", "prog.mcu"),
                            "caps": j.get("caps") or {}} for j in jobs]).encode()

    def enumerate_verdict_many_raw(self, payload: bytes, rank: int = 0, world: int = 1) -> str:
        """hgrd_gpu_enumerate_verdict_many_json as is: jobs JSON in, report
        JSON text out."""
        out = ctypes.c_void_p()
        rc = self._lib.hgrd_gpu_enumerate_verdict_many_json(self._ctx, payload, rank, world,
                                                            ctypes.byref(out))
        s = _take_string(self._lib, out)
        if rc != 0:
            raise RuntimeError(f"enumerate_verdict_many failed ({rc}): {s}")
        return s

    def enumerate_verdict_many(self, jobs, rank: int = 0, world: int = 1) -> List[dict]:
        """Many programs' sweeps at once (BASELINE config 5): jobs is a list
        of {"source", "file", "caps"}; returns per job its enumerateVerdict
        result (world 1) or this rank's sweep shard (parallel.merge_shards)."""
        return json.loads(self.enumerate_verdict_many_raw(self.sweep_jobs_payload(jobs), rank,
                                                          world))

    def enumerate_verdict(self, source: str, caps=None, file_name: str = "prog.mcu") -> dict:
        out = ctypes.c_void_p()
        rc = self._lib.hgrd_gpu_enumerate_verdict_json(self._ctx, source.encode(),
                                                       file_name.encode(),
                                                       _cfg_json(caps).encode(),
                                                       ctypes.byref(out))
        s = _take_string(self._lib, out)
        if rc != 0:
            raise RuntimeError(f"enumerate_verdict failed ({rc}): {s}")
        return json.loads(s)

    # -- instrumentation --
    def set_profiling(self, on: bool = True):
        self._lib.hgrd_gpu_set_profiling(self._ctx, 1 if on else 0)

    def last_profile(self) -> List[dict]:
        """[{name, ms}] per pipeline stage of the last check (CUDA events)."""
        return json.loads(self._lib.hgrd_gpu_last_profile(self._ctx).decode() or "[]")

    def set_fused(self, on: bool = True):
        """Enable (default) / disable the fused block-local check."""
        self._lib.hgrd_gpu_set_fused(self._ctx, 1 if on else 0)

    def set_jit(self, mode: int = 1):
        """NVRTC specialisation: 0 off, 1 auto (>= 2^14 threads), 2 always."""
        self._lib.hgrd_gpu_set_jit(self._ctx, mode)

    def jit_info(self) -> dict:
        return json.loads(self._lib.hgrd_gpu_jit_info(self._ctx).decode())

    def kernel_launches(self) -> int:
        return int(self._lib.hgrd_gpu_kernel_launches(self._ctx))

    def transfer_bytes(self):
        """(host->device, device->host) bytes copied by this context so far."""
        h, d = ctypes.c_ulonglong(), ctypes.c_ulonglong()
        rc = self._lib.hgrd_gpu_transfer_bytes(self._ctx, ctypes.byref(h), ctypes.byref(d))
        if rc:
            self._err("transfer_bytes", rc)
        return int(h.value), int(d.value)

    # -- device buffers --
    def reset(self):
        rc = self._lib.hgrd_gpu_buffers_reset(self._ctx)
        if rc:
            self._err("buffers_reset", rc)

    def alloc(self, elems: int) -> int:
        h = c_int32()
        rc = self._lib.hgrd_gpu_buffer_alloc(self._ctx, elems, ctypes.byref(h))
        if rc:
            self._err("buffer_alloc", rc)
        return h.value

    def write(self, handle: int, array, offset: int = 0):
        """array: contiguous int64 numpy array (host buffer)."""
        rc = self._lib.hgrd_gpu_buffer_write(self._ctx, handle, offset, int(array.size),
                                             array.ctypes.data)
        if rc:
            self._err("buffer_write", rc)

    def write_async(self, handle: int, array, offset: int = 0):
        """write() on the context's copy stream (hgrd_gpu_buffer_write_async):
        returns at once; the next check that uses the buffer waits for the
        copy on the device.  Keep `array` alive (and pinned, for overlap)
        until then."""
        rc = self._lib.hgrd_gpu_buffer_write_async(self._ctx, handle, offset, int(array.size),
                                                   array.ctypes.data)
        if rc:
            self._err("buffer_write_async", rc)

    def read(self, handle: int, out, offset: int = 0):
        rc = self._lib.hgrd_gpu_buffer_read(self._ctx, handle, offset, int(out.size),
                                            out.ctypes.data)
        if rc:
            self._err("buffer_read", rc)
        return out

    # -- sharded single-launch check (parallel.check_launch_sharded) --
    def shard_check(self, spec: LaunchSpec, block_begin: int, block_end: int):
        """INTRA races + counters of blocks [block_begin, block_end) and the
        shard's INTER summary tables (device).  Raises NotShardable."""
        res, races, traps = spec.new_result(0)
        sh = Shard(block_begin, block_end, None, None, 0)
        rc = self._lib.hgrd_gpu_shard_check(self._ctx, ctypes.byref(spec.launch),
                                            ctypes.byref(sh), ctypes.byref(res))
        if rc == HGRD_GPU_ENOTSUP:
            raise NotShardable(self._lib.hgrd_gpu_last_error(self._ctx).decode())
        if rc:
            self._err("shard_check", rc)
        return spec.decode(res), sh

    def shard_tables(self, sh: Shard, device: int = 0):
        """The shard's (lo, hi) INTER tables as int32 torch tensors sharing
        the context's device memory (for an in-place MIN / MAX all-reduce)."""
        import torch
        dev = torch.device("cuda", device)
        lo = torch.as_tensor(_CudaArray(sh.inter_lo, sh.inter_n), device=dev)
        hi = torch.as_tensor(_CudaArray(sh.inter_hi, sh.inter_n), device=dev)
        return lo, hi

    def stream(self) -> int:
        """The context's cudaStream_t (every kernel of the context runs on it)."""
        return int(self._lib.hgrd_gpu_stream(self._ctx) or 0)

    def wait_torch_stream(self, device: int = 0):
        """Order the context's stream after the work already queued on
        torch's current stream (a collective that produced its inputs)."""
        import torch
        cur = torch.cuda.current_stream(device)
        ext = torch.cuda.ExternalStream(self.stream(), device=torch.device("cuda", device))
        ext.wait_stream(cur)

    def shard_inter_scan(self, spec: LaunchSpec, lo, hi, elem_begin: int, n_elems: int,
                         device: int = 0):
        """Reduce-scatter variant, step 2a: per INTER key the minimum element
        of [elem_begin, elem_begin + n_elems) from the reduced tables `lo` /
        `hi` (int32 CUDA tensors of n_elems * n_sites entries, produced on
        torch's current stream — the context's stream waits for it).
        Returns uint64 numpy [3 * n_locs^2], 2^64 - 1 where none."""
        import numpy as np
        n_locs = max(len(spec.lowered["locs"]), 1)
        ke = np.zeros(3 * n_locs * n_locs, dtype=np.uint64)
        if n_elems:
            self.wait_torch_stream(device)
        rc = self._lib.hgrd_gpu_shard_inter_scan(
            self._ctx, ctypes.byref(spec.launch), lo.data_ptr() if n_elems else None,
            hi.data_ptr() if n_elems else None, elem_begin, n_elems,
            ke.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), len(ke))
        if rc == HGRD_GPU_ENOTSUP:
            raise NotShardable(self._lib.hgrd_gpu_last_error(self._ctx).decode())
        if rc:
            self._err("shard_inter_scan", rc)
        return ke

    def shard_inter_records(self, spec: LaunchSpec, sh: Shard, key_elem):
        """Step 2b: this shard's packed records of the realised INTER keys'
        first-found elements (`key_elem`: the MIN-reduced scan tables)."""
        import numpy as np
        key_elem = np.ascontiguousarray(key_elem, dtype=np.uint64)
        cap = 1 << 16
        while True:
            keys = np.zeros(cap, dtype=np.uint64)
            vals = np.zeros(cap, dtype=np.uint32)
            n = ctypes.c_uint64()
            rc = self._lib.hgrd_gpu_shard_inter_records(
                self._ctx, ctypes.byref(spec.launch), ctypes.byref(sh),
                key_elem.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), len(key_elem),
                keys.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                vals.ctypes.data_as(ctypes.POINTER(c_uint32)), cap, ctypes.byref(n))
            if rc == -7:  # E2BIG
                cap = max(cap * 2, int(n.value))
                continue
            if rc == HGRD_GPU_ENOTSUP:
                raise NotShardable(self._lib.hgrd_gpu_last_error(self._ctx).decode())
            if rc:
                self._err("shard_inter_records", rc)
            return keys[: n.value].copy(), vals[: n.value].copy()

    def shard_inter(self, spec: LaunchSpec, sh: Shard):
        """After the all-reduce: this shard's packed records of the realised
        INTER keys' first-found elements (numpy uint64 keys, uint32 vals)."""
        import numpy as np
        cap = 1 << 16
        while True:
            keys = np.zeros(cap, dtype=np.uint64)
            vals = np.zeros(cap, dtype=np.uint32)
            n = ctypes.c_uint64()
            rc = self._lib.hgrd_gpu_shard_inter(
                self._ctx, ctypes.byref(spec.launch), ctypes.byref(sh),
                keys.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                vals.ctypes.data_as(ctypes.POINTER(c_uint32)), cap, ctypes.byref(n))
            if rc == -7:  # E2BIG
                cap = max(cap * 2, int(n.value))
                continue
            if rc == HGRD_GPU_ENOTSUP:
                raise NotShardable(self._lib.hgrd_gpu_last_error(self._ctx).decode())
            if rc:
                self._err("shard_inter", rc)
            return keys[: n.value].copy(), vals[: n.value].copy()

    def shard_detect(self, spec: LaunchSpec, keys, vals) -> dict:
        """INTER-BLOCK races (with witnesses) of records gathered from all shards."""
        import numpy as np
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        vals = np.ascontiguousarray(vals, dtype=np.uint32)
        res, races, traps = spec.new_result(0)
        rc = self._lib.hgrd_gpu_shard_detect(
            self._ctx, ctypes.byref(spec.launch),
            keys.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
            vals.ctypes.data_as(ctypes.POINTER(c_uint32)), len(keys), ctypes.byref(res))
        if rc:
            self._err("shard_detect", rc)
        return spec.decode(res)

    def check_launch(self, spec: LaunchSpec, trap_cap: int = 256, raw: bool = False):
        res, races, traps = spec.new_result(trap_cap)
        rc = self._lib.hgrd_gpu_check_launch(self._ctx, ctypes.byref(spec.launch),
                                             ctypes.byref(res))
        if rc:
            self._err("check_launch", rc)
        return res if raw else spec.decode(res)


__all__ = ["ExecConfig", "SweepCaps", "GpuContext", "LaunchSpec", "Shard", "NotShardable",
           "count_inputs", "lower",
           "load_library", "LIBRARY_PATH", "RACE_KINDS", "LAUNCH_SEQUENTIAL",
           "LAUNCH_PAIRWISE", "LAUNCH_NO_WITNESS", "LAUNCH_GENERAL"]
