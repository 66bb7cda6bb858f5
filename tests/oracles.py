"""Test-side access to the CPU checkers under oracle/_ref (test infrastructure).

* ``RefOracle``  — the UNMODIFIED reference oracle (libhgrd_ref.so, built from
  /root/reference by oracle/Makefile).
* ``CpuOracle``  — the CPU restatement (libhgrd_oracle.so: oracle/cpu_oracle.cpp
  behind the shared host front end), which also reports witnesses and can
  check a single launch descriptor.

Only tests, __graft_entry__.smoke() and bench.py's CPU-baseline leg use these.
"""
from __future__ import annotations

import ctypes
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libhgrd_ref.so")
ORACLE_LIB = os.path.join(ROOT, "oracle", "_ref", "libhgrd_oracle.so")


def _cfg(cfg) -> bytes:
    if cfg is None:
        return b"{}"
    if isinstance(cfg, (bytes, str)):
        return cfg if isinstance(cfg, bytes) else cfg.encode()
    if isinstance(cfg, dict):
        return json.dumps(cfg).encode()
    return cfg.to_json().encode()


class RefOracle:
    def __init__(self, path: str = REF_LIB):
        self.lib = ctypes.CDLL(path)
        self.lib.hgrd_ref_run_concrete.restype = ctypes.c_void_p
        self.lib.hgrd_ref_run_concrete.argtypes = [ctypes.c_char_p] * 3
        self.lib.hgrd_ref_enumerate_verdict.restype = ctypes.c_void_p
        self.lib.hgrd_ref_enumerate_verdict.argtypes = [ctypes.c_char_p] * 3
        self.lib.hgrd_ref_free.argtypes = [ctypes.c_void_p]
        self.lib.hgrd_ref_analyze.restype = ctypes.c_void_p
        self.lib.hgrd_ref_analyze.argtypes = [ctypes.c_char_p] * 3
        self.lib.hgrd_ref_time_sweeps.restype = ctypes.c_double
        self.lib.hgrd_ref_time_sweeps.argtypes = [ctypes.c_void_p] * 3 + [
            ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        self.lib.hgrd_ref_time_parallel.restype = ctypes.c_double
        self.lib.hgrd_ref_time_parallel.argtypes = [ctypes.c_char_p] * 3 + [
            ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]

    def analyze(self, source: str, opts=None, file_name: str = "prog.mcu") -> dict:
        """The reference's static analyzer (analyzeProgram): race entries."""
        return self._take(self.lib.hgrd_ref_analyze(source.encode(), file_name.encode(),
                                                    _cfg(opts)))

    def time_sweeps(self, jobs, threads: int):
        """Wall seconds of enumerateVerdict over `jobs` [(source, file, caps)]
        on `threads` host threads; returns (seconds, total sweep races)."""
        n = len(jobs)
        arr = ctypes.c_char_p * max(n, 1)
        srcs = arr(*[j[0].encode() for j in jobs])
        files = arr(*[j[1].encode() for j in jobs])
        caps = arr(*[_cfg(j[2]) for j in jobs])
        races = ctypes.c_int(0)
        secs = self.lib.hgrd_ref_time_sweeps(srcs, files, caps, n, threads, ctypes.byref(races))
        return secs, races.value

    def _take(self, p) -> dict:
        s = ctypes.string_at(p).decode()
        self.lib.hgrd_ref_free(p)
        return json.loads(s)

    def run_concrete(self, source: str, config=None, file_name: str = "prog.mcu") -> dict:
        return self._take(self.lib.hgrd_ref_run_concrete(source.encode(), file_name.encode(),
                                                         _cfg(config)))

    def enumerate_verdict(self, source: str, caps=None, file_name: str = "prog.mcu") -> dict:
        return self._take(self.lib.hgrd_ref_enumerate_verdict(source.encode(),
                                                              file_name.encode(), _cfg(caps)))

    def time_parallel(self, source: str, config, threads: int, reps: int = 1,
                      file_name: str = "prog.mcu"):
        n = ctypes.c_int(-1)
        secs = self.lib.hgrd_ref_time_parallel(source.encode(), file_name.encode(), _cfg(config),
                                               threads, reps, ctypes.byref(n))
        return secs, n.value


class CpuOracle:
    def __init__(self, path: str = ORACLE_LIB):
        self.lib = ctypes.CDLL(path)
        P = ctypes.c_void_p
        for fn in ("hgrd_oracle_run_concrete_json", "hgrd_oracle_enumerate_verdict_json",
                   "hgrd_oracle_enumerate_verdict_batched_json"):
            getattr(self.lib, fn).argtypes = [ctypes.c_char_p] * 3 + [ctypes.POINTER(P)]
        self.lib.hgrd_oracle_free.argtypes = [P]
        self.lib.hgrd_oracle_enumerate_verdict_many_json.argtypes = [
            ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(P)]
        self.lib.hgrd_oracle_check_launch.argtypes = [P, P, P, ctypes.c_int32, P]
        self.lib.hgrd_oracle_sweep_shard_json.argtypes = [ctypes.c_char_p] * 3 + [
            ctypes.c_int, ctypes.c_int, ctypes.POINTER(P)]

    def _call(self, fn, source, cfg, file_name) -> dict:
        out = ctypes.c_void_p()
        rc = getattr(self.lib, fn)(source.encode(), file_name.encode(), _cfg(cfg),
                                   ctypes.byref(out))
        s = ctypes.string_at(out.value).decode()
        self.lib.hgrd_oracle_free(out)
        d = json.loads(s)
        if rc != 0:
            raise RuntimeError(f"{fn} failed ({rc}): {d}")
        return d

    def run_concrete(self, source: str, config=None, file_name: str = "prog.mcu") -> dict:
        return self._call("hgrd_oracle_run_concrete_json", source, config, file_name)

    def enumerate_verdict(self, source: str, caps=None, file_name: str = "prog.mcu") -> dict:
        return self._call("hgrd_oracle_enumerate_verdict_json", source, caps, file_name)

    def enumerate_verdict_batched(self, source: str, caps=None,
                                  file_name: str = "prog.mcu") -> dict:
        """The product's speculative batched sweep (host.cpp
        enumerateVerdictBatched) with the restatement as its batch backend."""
        return self._call("hgrd_oracle_enumerate_verdict_batched_json", source, caps, file_name)

    def enumerate_verdict_many(self, jobs, rank: int = 0, world: int = 1,
                               batched: bool = True) -> list:
        """sweepManyJson over [{"source", "file", "caps"}] (the product's
        many-sweeps path) with the restatement as backend."""
        out = ctypes.c_void_p()
        rc = self.lib.hgrd_oracle_enumerate_verdict_many_json(
            json.dumps(jobs).encode(), rank, world, 1 if batched else 0, ctypes.byref(out))
        s = ctypes.string_at(out.value).decode()
        self.lib.hgrd_oracle_free(out)
        if rc != 0:
            raise RuntimeError(f"enumerate_verdict_many failed ({rc}): {s}")
        return json.loads(s)

    def sweep_shard(self, source: str, caps=None, file_name: str = "prog.mcu",
                    rank: int = 0, world: int = 1) -> dict:
        out = ctypes.c_void_p()
        rc = self.lib.hgrd_oracle_sweep_shard_json(source.encode(), file_name.encode(),
                                                    _cfg(caps), rank, world, ctypes.byref(out))
        s = ctypes.string_at(out.value).decode()
        self.lib.hgrd_oracle_free(out)
        if rc != 0:
            raise RuntimeError(f"sweep_shard failed ({rc}): {s}")
        return json.loads(s)

    def check_launch(self, spec, buffers, trap_cap: int = 256) -> dict:
        """Check one LaunchSpec against int64 numpy buffers (handle = list index)."""
        n = len(buffers)
        ptrs = (ctypes.c_void_p * max(n, 1))(*[b.ctypes.data for b in buffers])
        sizes = (ctypes.c_int64 * max(n, 1))(*[b.size for b in buffers])
        res, races, traps = spec.new_result(trap_cap)
        rc = self.lib.hgrd_oracle_check_launch(ctypes.byref(spec.launch), ptrs, sizes, n,
                                               ctypes.byref(res))
        if rc != 0:
            raise RuntimeError(f"oracle check_launch failed ({rc})")
        return spec.decode(res)


def strip_extras(result: dict) -> dict:
    """Drop the fields the reference does not have (witnesses, stats)."""
    return {k: v for k, v in result.items() if k not in ("witnesses", "stats", "configs")}
