"""Seeded synthetic workloads (shared by the oracle side and the CUDA side).

No method arithmetic lives here (see synth/gen.py for the definition). Three
independent implementations of one definition:
  * ``synth.gen``            numpy (reference definition, any size that fits RAM)
  * ``libsynth.so``          host C, threaded (streams c4's 2^33 doubles to the oracle)
  * ``libsynth_cuda.so``     device kernels (bench.py fills HBM directly)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import gen
from .gen import CONFIGS

_HERE = os.path.dirname(os.path.abspath(__file__))
_HOST_SO = os.path.join(_HERE, "libsynth.so")
_CUDA_SO = os.path.join(_HERE, "libsynth_cuda.so")
NVCC_ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def build(cuda: bool = True) -> None:
    """Compile libsynth.so (gcc) and, if requested, libsynth_cuda.so (nvcc, sm_100a)."""
    src = os.path.join(_HERE, "gen.c")
    if _stale(_HOST_SO, [src]):
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-pthread", src, "-o", _HOST_SO])
    if cuda:
        cus = [os.path.join(_HERE, "csrc", f) for f in ("gen.cu", "probe.cu")]
        if _stale(_CUDA_SO, cus):
            subprocess.check_call(["nvcc", *NVCC_ARCH, "-O3", "-lineinfo", "-Xcompiler", "-fPIC",
                                   "-shared", *cus, "-o", _CUDA_SO])


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


_host = None
_cuda = None


def host_lib():
    global _host
    if _host is None:
        if not os.path.exists(_HOST_SO):
            build(cuda=False)
        lib = ctypes.CDLL(_HOST_SO)
        u64, i32, p = ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
        lib.synth_uniform.argtypes = [p, u64, u64, u64, u64, i32, i32, i32]
        lib.synth_cancel_unpermuted.argtypes = [p, u64, u64, u64, u64, i32, i32, i32, i32, i32]
        lib.synth_keys.argtypes = [p, u64, u64, u64, u64, i32]
        for f in (lib.synth_uniform, lib.synth_cancel_unpermuted, lib.synth_keys):
            f.restype = None
        _host = lib
    return _host


def cuda_lib():
    global _cuda
    if _cuda is None:
        if not os.path.exists(_CUDA_SO):
            raise RuntimeError(f"{_CUDA_SO} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(_CUDA_SO)
        u64, i32, p = ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
        lib.synth_gpu_uniform.argtypes = [p, u64, u64, u64, u64, i32, i32, p]
        lib.synth_gpu_cancel_unpermuted.argtypes = [p, u64, u64, u64, u64, i32, i32, i32, i32, p]
        lib.synth_gpu_keys_signed.argtypes = [p, u64, u64, u64, u64, p]
        lib.synth_probe_read.argtypes = [p, u64, p, i32, i32, i32, p]
        lib.synth_gpu_fill_after_trigger.argtypes = [p, u64, ctypes.c_double, ctypes.c_longlong, p]
        lib.synth_gpu_fill_after_trigger.restype = ctypes.c_int
        lib.synth_probe_read.restype = ctypes.c_int
        for f in (lib.synth_gpu_uniform, lib.synth_gpu_cancel_unpermuted, lib.synth_gpu_keys_signed):
            f.restype = ctypes.c_int
        _cuda = lib
    return _cuda


def _threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def host_generate(name: str, start: int = 0, count: int | None = None, out: np.ndarray | None = None,
                  nthreads: int | None = None) -> np.ndarray:
    """Elements [start, start+count) of config ``name`` via the threaded C generator.
    c3 is returned in PRE-permutation order (the exact sum does not depend on order)."""
    cfg = CONFIGS[name]
    if count is None:
        count = cfg["n"] - start
    if start < 0 or start + count > cfg["n"]:
        raise ValueError("range outside config")
    if out is None:
        out = np.empty(count, dtype=np.float64)
    assert out.dtype == np.float64 and out.size >= count and out.flags.c_contiguous
    nt = nthreads or _threads()
    lib = host_lib()
    ptr = out.ctypes.data
    if cfg["kind"] == "cancel":
        lib.synth_cancel_unpermuted(ptr, start, count, cfg["seed"], cfg["npairs"], cfg["pair_lo"],
                                    cfg["pair_hi"], cfg["tiny_lo"], cfg["tiny_hi"], nt)
    else:
        lib.synth_uniform(ptr, start, count, cfg["seed"], cfg["st"], cfg["lo"], cfg["hi"], nt)
    return out[:count]


def host_bits(name: str, start: int = 0, count: int | None = None) -> np.ndarray:
    """Elements [start, start+count) of a "bits" config (other input formats) as bit patterns,
    the draws from the threaded C generator (gen.bits is the numpy definition)."""
    from .gen import bits_fix
    cfg = CONFIGS[name]
    if count is None:
        count = cfg["n"] - start
    return bits_fix(host_keys(cfg["seed"], cfg["st"], start, count), cfg["fmt"])


def device_bits(name: str, device=None):
    """A "bits" config as a CUDA tensor of its format (float32 / float16 / bfloat16)."""
    import torch
    cfg = CONFIGS[name]
    b = host_bits(name)
    t = torch.from_numpy(b.view(np.int32 if cfg["fmt"] == "f32" else np.int16)).to(
        torch.device(device if device is not None else "cuda"))
    return t.view({"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}[cfg["fmt"]])


def csr_offsets(name: str, device=None):
    """int64 CUDA tensor of a "csr" config's offsets."""
    import torch
    from .gen import csr_offsets as offs
    return torch.from_numpy(offs(CONFIGS[name])).to(torch.device(device if device is not None else "cuda"))


def host_keys(seed: int, st: int, start: int, count: int, nthreads: int | None = None) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    host_lib().synth_keys(out.ctypes.data, start, count, seed, st, nthreads or _threads())
    return out


def device_generate(name: str, start: int = 0, count: int | None = None, device=None,
                    permute: bool = True, out=None):
    """Elements [start, start+count) of config ``name`` as a float64 CUDA tensor.

    c3 (whole array only when ``permute``) is permuted by a stable sort of the
    positions on their keys U(3, 2, idx) - input preparation, not the timed path."""
    import torch

    cfg = CONFIGS[name]
    if count is None:
        count = cfg["n"] - start
    if start < 0 or start + count > cfg["n"]:
        raise ValueError("range outside config")
    dev = torch.device(device if device is not None else "cuda")
    stream = torch.cuda.current_stream(dev).cuda_stream
    lib = cuda_lib()
    if out is None:
        out = torch.empty(count, dtype=torch.float64, device=dev)
    if cfg["kind"] == "cancel":
        rc = lib.synth_gpu_cancel_unpermuted(out.data_ptr(), start, count, cfg["seed"], cfg["npairs"],
                                             cfg["pair_lo"], cfg["pair_hi"], cfg["tiny_lo"],
                                             cfg["tiny_hi"], stream)
        if rc:
            raise RuntimeError(f"synth_gpu_cancel_unpermuted failed: {rc}")
        if permute:
            if start != 0 or count != cfg["n"]:
                raise ValueError("permuted c3 is only available whole")
            keys = torch.empty(count, dtype=torch.int64, device=dev)
            rc = lib.synth_gpu_keys_signed(keys.data_ptr(), 0, count, cfg["seed"], 2, stream)
            if rc:
                raise RuntimeError(f"synth_gpu_keys_signed failed: {rc}")
            _, perm = torch.sort(keys, stable=True)
            del keys
            out = out.index_select(0, perm)
            del perm
    else:
        rc = lib.synth_gpu_uniform(out.data_ptr(), start, count, cfg["seed"], cfg["st"], cfg["lo"],
                                   cfg["hi"], stream)
        if rc:
            raise RuntimeError(f"synth_gpu_uniform failed: {rc}")
    return out


def probe_read_gbs(x, variant: int = 0, blocks: int = 148, threads: int = 512, reps: int = 20) -> float:
    """Read bandwidth (GB/s, median of reps, CUDA events) of probe `variant` over tensor x."""
    import statistics

    import torch
    out = torch.empty(blocks * threads, dtype=torch.int32, device=x.device)
    st = torch.cuda.current_stream(x.device)
    lib = cuda_lib()
    nbytes = x.numel() * x.element_size()
    for _ in range(3):
        lib.synth_probe_read(x.data_ptr(), nbytes, out.data_ptr(), variant, blocks, threads, st.cuda_stream)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        rc = lib.synth_probe_read(x.data_ptr(), nbytes, out.data_ptr(), variant, blocks, threads, st.cuda_stream)
        b.record(st)
        b.synchronize()
        if rc:
            raise RuntimeError(f"probe {variant} failed: {rc}")
        ts.append(a.elapsed_time(b))
    return nbytes / statistics.median(ts) / 1e6
