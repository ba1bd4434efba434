"""Exact floating-point summation on B200 (sm_100a): Python binding of libxsum.so.

A thin ctypes layer over the C-ABI in ``include/xsum.h`` (same names, argument
marshalling only). PyTorch supplies device memory and streams; every arithmetic
step of the summation runs in the library's CUDA kernels. There is no CPU
fallback: if ``libxsum.so`` is missing or no CUDA device is present, calls raise.

Method: Goodrich & Eldawy, "Parallel Algorithms for Summing Floating-Point
Numbers" (arXiv 1605.05436); see DESIGN.md for the mapping of the paper's steps
to kernels and include/xsum.h for the boundary.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "libxsum.so")
# development only: an alternative build of the same C-ABI (tools/variants.py, the checked build of
# tools/checked_build.py) is loaded only when XSUM_DEV=1 is set as well, so a stray XSUM_LIBRARY
# cannot silently swap the library under test
if os.environ.get("XSUM_DEV") == "1" and os.environ.get("XSUM_LIBRARY"):
    SO_PATH = os.environ["XSUM_LIBRARY"]

STATE_BYTES = 384
RESULT_BYTES = 48
CANON_LIMBS = 34
RADIX_BITS = 52
NDIGITS = 42
MAGIC = 0x4D555358
VERSION = 1
F_NAN, F_PINF, F_NINF, F_OVERFLOW, F_INEXACT, F_MISMATCH = 1, 2, 4, 8, 16, 32
F_OVERFLOW32, F_INEXACT32 = 64, 128
F_PEER_TIMEOUT = 256
F_CAPACITY = 512
TOP_DIGIT_MAX = 1 << 29

OK, EINVAL, ECAPACITY, ECUDA, EMISMATCH, ENOMEM = range(6)

# sparse state image (include/xsum.h): 24-byte header + nnz records (digit << 6) | index
SPARSE_MAGIC = 0x41505358
SPARSE_HEADER_BYTES = 24
SEG_LANES_MAX = 256          # segments of at most this many elements are summed one lane each
SPARSE_MAX_BYTES = SPARSE_HEADER_BYTES + 8 * NDIGITS

# every entry point declared in include/xsum.h
EXPORTS = ("xsum_state_bytes", "xsum_scratch_bytes", "xsum_result_bytes", "xsum_create", "xsum_reset",
           "xsum_accumulate", "xsum_accumulate_host", "xsum_merge", "xsum_finalize_round", "xsum_sum",
           "xsum_destroy", "xsum_count", "xsum_sum_segments", "xsum_sum_segments_csr", "xsum_status_str",
           "xsum_launch_count", "xsum_set_grid_limit", "xsum_accumulate_f32", "xsum_sum_f32", "xsum_merge_round",
           "xsum_accumulate_f16", "xsum_accumulate_bf16", "xsum_sum_f16", "xsum_sum_bf16",
           "xsum_to_sparse", "xsum_merge_sparse", "xsum_peer_buffer_bytes", "xsum_sum_allreduce",
           "xsum_peer_selftest", "xsum_sum_segments_ex", "xsum_accumulate_host_ex", "xsum_save_state",
           "xsum_check_state_image", "xsum_load_state", "xsum_sum_strided_work_bytes", "xsum_sum_strided",
           "xsum_sum_segments_ws", "xsum_sum_segments_csr_lanes", "xsum_condsens_work_bytes", "xsum_sum_condsens")


class XsumError(RuntimeError):
    def __init__(self, fn: str, status: int):
        self.status = status
        super().__init__(f"{fn} failed: {status_str(status)} ({status})")


_lib = None


def build(force: bool = False) -> str:
    """Compile libxsum.so in-tree (nvcc, sm_100a)."""
    import importlib
    return importlib.import_module(__name__ + "._build").build(force=force)


def lib() -> ctypes.CDLL:
    """Load libxsum.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise RuntimeError(f"{SO_PATH} not built: run `python -m paper_1605_05436_b200._build` "
                               "or __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(SO_PATH)
        p, u64, u32, i32, sz = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_size_t
        sig = {
            "xsum_state_bytes": ([], sz), "xsum_scratch_bytes": ([i32], sz), "xsum_result_bytes": ([], sz),
            "xsum_create": ([ctypes.POINTER(p), i32, p, p, sz, p], i32), "xsum_reset": ([p, p], i32),
            "xsum_accumulate": ([p, p, u64, p], i32), "xsum_accumulate_host": ([p, p, u64, p, sz, p], i32),
            "xsum_merge": ([p, p, u32, p], i32), "xsum_finalize_round": ([p, p, p, p], i32),
            "xsum_sum": ([p, p, u64, p, p, p], i32), "xsum_destroy": ([p], i32), "xsum_count": ([p], u64),
            "xsum_sum_segments": ([p, u64, u64, p, p, p, p], i32),
            "xsum_sum_segments_csr": ([p, p, u64, p, p, p, p], i32),
            "xsum_status_str": ([i32], ctypes.c_char_p), "xsum_launch_count": ([], u64),
            "xsum_set_grid_limit": ([p, u32], i32),
            "xsum_accumulate_f32": ([p, p, u64, p], i32), "xsum_sum_f32": ([p, p, u64, p, p, p], i32),
            "xsum_merge_round": ([p, p, u32, p, p, p], i32),
            "xsum_accumulate_f16": ([p, p, u64, p], i32), "xsum_accumulate_bf16": ([p, p, u64, p], i32),
            "xsum_sum_f16": ([p, p, u64, p, p, p], i32), "xsum_sum_bf16": ([p, p, u64, p, p, p], i32),
            "xsum_to_sparse": ([p, p, p, p], i32), "xsum_merge_sparse": ([p, p, p, u32, p], i32),
            "xsum_peer_buffer_bytes": ([u32], sz),
            "xsum_sum_allreduce": ([p, p, u64, p, u32, u32, u64, p, p, p], i32),
            "xsum_peer_selftest": ([p, p, u32, u64, p, p, p], i32),
            "xsum_sum_segments_ex": ([p, i32, u64, u64, p, p, p, p, p, p], i32),
            "xsum_accumulate_host_ex": ([p, p, u64, i32, p, sz, p], i32),
            "xsum_save_state": ([p, p, p], i32), "xsum_check_state_image": ([p], i32),
            "xsum_load_state": ([p, p, p], i32),
            "xsum_sum_strided_work_bytes": ([u64, u64, u64, i32], sz),
            "xsum_sum_strided": ([p, i32, u64, u64, u64, p, p, p, p, sz, p], i32),
            "xsum_sum_segments_ws": ([p, i32, u64, u64, p, p, p, p, p, p, p], i32),
            "xsum_sum_segments_csr_lanes": ([p, i32, u64, p, p, p, p, p, p, p], i32),
            "xsum_condsens_work_bytes": ([u64], sz),
            "xsum_sum_condsens": ([p, u64, i32, p, sz, p, p, p, p], i32),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def check_state_image(image: bytes) -> bool:
    """Host-side validation of a 384-byte state image (xsum_check_state_image): header, flags,
    count and digit ranges. True if the image is a valid checkpoint."""
    image = bytes(image)
    return len(image) == STATE_BYTES and lib().xsum_check_state_image(image) == 0


def status_str(s: int) -> str:
    try:
        return lib().xsum_status_str(s).decode()
    except Exception:  # pragma: no cover
        return "?"


def _check(fn: str, status: int) -> None:
    if status != OK:
        raise XsumError(fn, status)


def launch_count() -> int:
    return int(lib().xsum_launch_count())


@dataclass(frozen=True)
class Result:
    """Host copy of ``xsum_result`` (include/xsum.h)."""
    value: float
    bits: int
    direction: int
    flags: int
    msb_exp: int | None
    sign: int
    count: int
    sig53: int
    exp2: int
    bits_f32: int        # bits of the RN-even binary32 rounding of the exact sum

    @property
    def value_f32(self) -> float:
        return float(np.array([self.bits_f32], dtype=np.uint32).view(np.float32)[0])

    @staticmethod
    def from_bytes(b: bytes | np.ndarray) -> "Result":
        a = np.frombuffer(bytes(b), dtype=np.uint8)
        assert a.size == RESULT_BYTES
        value = float(a[0:8].view(np.float64)[0])
        bits = int(a[0:8].view(np.uint64)[0])
        i32 = a[8:24].view(np.int32)
        u32 = a[8:24].view(np.uint32)
        count = int(a[24:32].view(np.uint64)[0])
        sig53 = int(a[32:40].view(np.uint64)[0])
        exp2 = int(a[40:44].view(np.int32)[0])
        b32 = int(a[44:48].view(np.uint32)[0])
        msb = int(i32[2])
        return Result(value=value, bits=bits, direction=int(i32[0]), flags=int(u32[1]),
                      msb_exp=None if msb == -(2 ** 31) else msb, sign=int(i32[3]), count=count,
                      sig53=sig53, exp2=exp2, bits_f32=b32)


def _torch():
    import torch
    return torch


def _stream_ptr(device) -> int:
    """The current CUDA stream of `device` as a raw cudaStream_t value (no Stream object)."""
    torch = _torch()
    idx = device.index if isinstance(device, torch.device) else device
    if idx is None:
        idx = torch.cuda.current_device()
    return torch._C._cuda_getCurrentRawStream(idx)


def _as_f64_cuda(t, allow_f32: bool = False):
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("expected a CUDA tensor")
    ok = (torch.float64, torch.float32, torch.float16, torch.bfloat16) if allow_f32 else (torch.float64,)
    if t.dtype not in ok:
        raise TypeError(f"expected one of {ok}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t


def _is_f32(t) -> bool:
    return t.dtype == _torch().float32


# per input dtype: (accumulate entry point, fused sum entry point)
_ENTRY = {"float64": ("xsum_accumulate", "xsum_sum"), "float32": ("xsum_accumulate_f32", "xsum_sum_f32"),
          "float16": ("xsum_accumulate_f16", "xsum_sum_f16"), "bfloat16": ("xsum_accumulate_bf16", "xsum_sum_bf16")}


_FNS: dict = {}


def _fns_for(t):
    """(accumulate fn, fused-sum fn, names) of the library for a CUDA tensor's dtype; the hot
    per-call path (one dict lookup instead of string work)."""
    f = _FNS.get(t.dtype)
    if f is None:
        torch = _torch()
        if not isinstance(t, torch.Tensor):
            raise TypeError("expected a CUDA tensor")
        key = str(t.dtype).replace("torch.", "")
        if key not in _ENTRY:
            raise TypeError(f"expected float64 / float32 / float16 / bfloat16, got {t.dtype}")
        a, s_ = _ENTRY[key]
        f = _FNS[t.dtype] = (getattr(lib(), a), getattr(lib(), s_), a, s_)
    if not t.is_cuda:
        raise TypeError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return f


class Accumulator:
    """An exact superaccumulator living in device memory (the xsum_ctx handle).

    ``add`` streams device tensors into it, ``add_host`` host arrays, ``merge``
    other accumulators' state images (e.g. the all-gather of the per-GPU states),
    ``result`` rounds it. All calls are asynchronous on the current stream except
    the ones that return host values."""

    def __init__(self, device=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1605_05436_b200 needs a CUDA device (no CPU fallback)")
        self.device = torch.device(device if device is not None else "cuda", )
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        L = lib()
        self.state = torch.zeros(STATE_BYTES, dtype=torch.uint8, device=self.device)
        nscr = int(L.xsum_scratch_bytes(self.device.index))
        self.scratch = torch.zeros(nscr, dtype=torch.uint8, device=self.device)
        self._res = torch.zeros(RESULT_BYTES, dtype=torch.uint8, device=self.device)
        self._canon = torch.zeros(CANON_LIMBS, dtype=torch.int64, device=self.device)
        self._idx = self.device.index
        self._res_ptr, self._canon_ptr = self._res.data_ptr(), self._canon.data_ptr()
        self._stage = None
        self._host_refs = []
        h = ctypes.c_void_p()
        _check("xsum_create", L.xsum_create(ctypes.byref(h), self.device.index, self.state.data_ptr(),
                                            self.scratch.data_ptr(), nscr, _stream_ptr(self.device)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            try:
                _lib.xsum_destroy(h)
            except Exception:  # pragma: no cover
                pass
            self._h = None

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    @property
    def count(self) -> int:
        """Summands in the state (xsum_count; after a merge it waits for the merged count)."""
        c = int(lib().xsum_count(self._h))
        if c == (1 << 64) - 1:
            raise XsumError("xsum_count", ECUDA)
        return c

    def _on_device(self, t, what: str = "tensor"):
        if t.device.index != self._idx:
            raise ValueError(f"{what} is on {t.device}, the accumulator on {self.device}")
        return t

    def set_grid_limit(self, max_blocks: int) -> "Accumulator":
        """Cap the blocks of an accumulate launch (0 = one per SM)."""
        _check("xsum_set_grid_limit", lib().xsum_set_grid_limit(self._h, max_blocks))
        return self

    def reset(self) -> "Accumulator":
        _check("xsum_reset", lib().xsum_reset(self._h, _stream_ptr(self.device)))
        return self

    def add(self, x) -> "Accumulator":
        """Sum a float64 / float32 / float16 / bfloat16 CUDA tensor into the state, exactly."""
        fa, _, name, _ = _fns_for(x)
        if x.device.index != self._idx:
            self._on_device(x)
        rc = fa(self._h, x.data_ptr(), x.numel(), _stream_ptr(self._idx))
        if rc:
            raise XsumError(name, rc)
        return self

    def add_host(self, x, stage_bytes: int = 128 << 20) -> "Accumulator":
        """Sum a host array/tensor (float64, float32, float16 or bfloat16; pinned memory overlaps
        copy and compute) through double-buffered staging chunks (xsum_accumulate_host_ex)."""
        torch = _torch()
        if isinstance(x, np.ndarray):
            if x.dtype not in (np.float64, np.float32, np.float16):
                x = np.asarray(x, dtype=np.float64)
            x = torch.from_numpy(np.ascontiguousarray(x))
        if x.is_cuda or x.dtype not in (torch.float64, torch.float32, torch.float16, torch.bfloat16) or \
                not x.is_contiguous():
            raise TypeError("expected a contiguous host float64 / float32 / float16 / bfloat16 array")
        if self._stage is None or self._stage.numel() < stage_bytes:
            self._stage = torch.empty(stage_bytes, dtype=torch.uint8, device=self.device)
        _check("xsum_accumulate_host_ex", lib().xsum_accumulate_host_ex(
            self._h, x.data_ptr(), x.numel(), _DT[str(x.dtype).replace("torch.", "")], self._stage.data_ptr(),
            self._stage.numel(), _stream_ptr(self.device)))
        # keep every source alive until its copies are done: the stream waited for each chunk's
        # copy before accumulating it, so an event recorded on it now passes after the last copy
        # (torch's pinned-memory cache cannot see the library's raw copies)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        self._host_refs = [(e, t) for e, t in self._host_refs if not e.query()] + [(ev, x)]
        return self

    def merge(self, states) -> "Accumulator":
        """Add packed state images (uint8 CUDA tensor of k*384 bytes, or another Accumulator)."""
        torch = _torch()
        if isinstance(states, Accumulator):
            states = states.state
        if not (isinstance(states, torch.Tensor) and states.is_cuda and states.dtype == torch.uint8
                and states.is_contiguous() and states.numel() % STATE_BYTES == 0):
            raise TypeError("expected a contiguous uint8 CUDA tensor of k*384 bytes")
        self._on_device(states, "states")
        k = states.numel() // STATE_BYTES
        _check("xsum_merge", lib().xsum_merge(self._h, states.data_ptr(), k, _stream_ptr(self.device)))
        return self

    def save_state(self) -> bytes:
        """Checkpoint: the 384-byte state image after everything enqueued so far
        (xsum_save_state; synchronizes the stream)."""
        buf = ctypes.create_string_buffer(STATE_BYTES)
        _check("xsum_save_state", lib().xsum_save_state(self._h, buf, _stream_ptr(self.device)))
        return buf.raw

    def load_state(self, image: bytes) -> "Accumulator":
        """Resume: state := a checkpoint image (validated host-side first, xsum_load_state)."""
        image = bytes(image)
        if len(image) != STATE_BYTES:
            raise ValueError(f"a state image has {STATE_BYTES} bytes, got {len(image)}")
        _check("xsum_load_state", lib().xsum_load_state(self._h, image, _stream_ptr(self.device)))
        return self

    def save(self, path) -> None:
        """Write the checkpoint to `path` atomically (temporary file + rename)."""
        data = self.save_state()
        tmp = f"{path}.tmp{os.getpid()}"
        with open(tmp, "wb") as f:
            f.write(data)
            f.flush()
            os.fsync(f.fileno())
        os.replace(tmp, path)

    @classmethod
    def load(cls, path, device=None) -> "Accumulator":
        """A new accumulator resumed from the checkpoint file at `path`."""
        with open(path, "rb") as f:
            data = f.read()
        return cls(device).load_state(data)

    def merge_round(self, states, canon: bool = False, out=None):
        """state := sum of the packed state images, then round (one launch; xsum_merge_round).
        Returns the device (result, canon) like finalize_async; `out` (optional uint8 CUDA tensor
        of RESULT_BYTES) receives the result record instead of the accumulator's own buffer."""
        torch = _torch()
        if not (isinstance(states, torch.Tensor) and states.is_cuda and states.dtype == torch.uint8
                and states.is_contiguous() and states.numel() % STATE_BYTES == 0):
            raise TypeError("expected a contiguous uint8 CUDA tensor of k*384 bytes")
        self._on_device(states, "states")
        res = self._res if out is None else self._out(out)
        _check("xsum_merge_round", lib().xsum_merge_round(
            self._h, states.data_ptr(), states.numel() // STATE_BYTES, res.data_ptr(),
            self._canon.data_ptr() if canon else None, _stream_ptr(self.device)))
        return res, (self._canon if canon else None)

    def _out(self, out):
        torch = _torch()
        if not (isinstance(out, torch.Tensor) and out.is_cuda and out.dtype == torch.uint8 and out.is_contiguous()
                and out.numel() == RESULT_BYTES and out.data_ptr() % 8 == 0):
            raise TypeError("out must be a contiguous, 8-B aligned uint8 CUDA tensor of RESULT_BYTES")
        return self._on_device(out, "out")

    def sum_allreduce(self, x, bufs_dev: int, rank: int, world: int, epoch: int, canon: bool = False, out=None):
        """Fused multi-GPU step (xsum_sum_allreduce): state := exact sum of every rank's shard, in
        one launch per rank; `bufs_dev` is the device address of the array of the world exchange
        buffer pointers (dist.PeerExchange sets it up). Returns the device (result, canon); `out`
        as in merge_round."""
        x = self._on_device(_as_f64_cuda(x))
        res = self._res if out is None else self._out(out)
        _check("xsum_sum_allreduce", lib().xsum_sum_allreduce(
            self._h, x.data_ptr(), x.numel(), bufs_dev, rank, world, epoch, res.data_ptr(),
            self._canon.data_ptr() if canon else None, _stream_ptr(self.device)))
        return res, (self._canon if canon else None)

    def to_sparse(self):
        """Sparse image of the state (xsum_to_sparse): (uint8 CUDA tensor of SPARSE_MAX_BYTES,
        its valid byte count as a host int)."""
        torch = _torch()
        out = torch.zeros(SPARSE_MAX_BYTES, dtype=torch.uint8, device=self.device)
        nb = torch.zeros(1, dtype=torch.int32, device=self.device)
        _check("xsum_to_sparse", lib().xsum_to_sparse(self._h, out.data_ptr(), nb.data_ptr(),
                                                      _stream_ptr(self.device)))
        n = int(nb.item())
        return out[:n], n

    def merge_sparse(self, images, offsets) -> "Accumulator":
        """State += the sparse images in `images` (uint8 CUDA tensor) starting at byte
        `offsets` (int64 CUDA tensor, multiples of 8)."""
        torch = _torch()
        if not (isinstance(images, torch.Tensor) and images.is_cuda and images.dtype == torch.uint8 and
                images.is_contiguous()):
            raise TypeError("images must be a contiguous uint8 CUDA tensor")
        if not (isinstance(offsets, torch.Tensor) and offsets.is_cuda and offsets.dtype == torch.int64 and
                offsets.is_contiguous()):
            raise TypeError("offsets must be a contiguous int64 CUDA tensor")
        self._on_device(images, "images")
        self._on_device(offsets, "offsets")
        base = images if images.numel() else torch.zeros(8, dtype=torch.uint8, device=self.device)
        _check("xsum_merge_sparse", lib().xsum_merge_sparse(self._h, base.data_ptr(), offsets.data_ptr(),
                                                            offsets.numel(), _stream_ptr(self.device)))
        return self

    def finalize_async(self, canon: bool = False):
        """Enqueue the rounding; returns the (result bytes, canon limbs or None) device tensors."""
        _check("xsum_finalize_round", lib().xsum_finalize_round(
            self._h, self._res.data_ptr(), self._canon.data_ptr() if canon else None,
            _stream_ptr(self.device)))
        return self._res, (self._canon if canon else None)

    def result(self) -> Result:
        res, _ = self.finalize_async()
        return Result.from_bytes(res.cpu().numpy().tobytes())

    def exact(self) -> tuple[Result, np.ndarray]:
        """(rounded result, 34-limb two's complement image of the exact sum * 2^1074)."""
        res, canon = self.finalize_async(canon=True)
        return Result.from_bytes(res.cpu().numpy().tobytes()), canon.cpu().numpy().view(np.uint64).copy()

    def sum(self, x, canon: bool = False, out=None):
        """One-shot fused path (xsum_sum / xsum_sum_f32): state := sum(x); returns device
        (result, canon); `out` as in merge_round."""
        _, fs, _, name = _fns_for(x)
        if x.device.index != self._idx:
            self._on_device(x)
        res = self._res if out is None else self._out(out)
        rc = fs(self._h, x.data_ptr(), x.numel(), res.data_ptr(), self._canon_ptr if canon else None,
                _stream_ptr(self._idx))
        if rc:
            raise XsumError(name, rc)
        return res, (self._canon if canon else None)


CONDSENS_INFO_BYTES = 152


@dataclass(frozen=True)
class CondSensInfo:
    """Host copy of ``xsum_condsens_info`` (include/xsum.h): the last iteration of the
    condition-number-sensitive sum."""
    r: int
    iterations: int
    e_cut: int | None            # None: nothing was truncated
    exact: bool
    rule: int
    root: dict                   # {index: digit} of the root's r-truncated sparse superaccumulator

    @staticmethod
    def from_bytes(b) -> "CondSensInfo":
        a = np.frombuffer(bytes(b), dtype=np.uint8)
        assert a.size == CONDSENS_INFO_BYTES
        r, it = (int(v) for v in a[0:8].view(np.uint32))
        e_cut = int(a[8:12].view(np.int32)[0])
        exact, rule, nnz = (int(v) for v in a[12:24].view(np.uint32))
        rec = a[24:24 + 8 * 16].view(np.int64)[:nnz]
        return CondSensInfo(r=r, iterations=it, e_cut=None if e_cut < 0 else e_cut, exact=bool(exact), rule=rule,
                            root={int(v & 63): int(v >> 6) for v in rec})


def condsens_work_bytes(n: int) -> int:
    return int(lib().xsum_condsens_work_bytes(n))


def sum_condsens(x, rule: int = 1, canon: bool = False, work=None, res=None, info=None):
    """Condition-number-sensitive sum of a float64 CUDA tensor (xsum_sum_condsens):
    the r = 2, 4, 16 truncated iterations with a stopping condition (rule 1 or 2), then the exact
    pass if needed. Returns device tensors (result record, info record, canonical image of the
    truncated root or None); no host synchronization. `work` (uint8, >= condsens_work_bytes(n),
    256-B aligned), `res` and `info` may be passed in to reuse buffers."""
    torch = _torch()
    x = _as_f64_cuda(x)
    nb = condsens_work_bytes(x.numel())
    if work is None or work.numel() < nb:
        work = torch.empty(nb, dtype=torch.uint8, device=x.device)
    elif not (work.is_cuda and work.dtype == torch.uint8 and work.is_contiguous() and work.device == x.device
              and work.data_ptr() % 256 == 0):
        raise TypeError("work must be a contiguous, 256-B aligned uint8 CUDA tensor on x's device")
    if res is None:
        res = torch.empty(RESULT_BYTES, dtype=torch.uint8, device=x.device)
    if info is None:
        info = torch.empty(CONDSENS_INFO_BYTES, dtype=torch.uint8, device=x.device)
    for t, nbytes in ((res, RESULT_BYTES), (info, CONDSENS_INFO_BYTES)):
        if not (t.is_cuda and t.dtype == torch.uint8 and t.numel() == nbytes and t.is_contiguous()
                and t.data_ptr() % 8 == 0 and t.device == x.device):
            raise TypeError("res / info must be 8-B aligned uint8 CUDA tensors of their record size")
    cn = torch.empty(CANON_LIMBS, dtype=torch.int64, device=x.device) if canon else None
    xp = x if x.numel() else torch.zeros(1, dtype=torch.float64, device=x.device)
    with torch.cuda.device(x.device):
        _check("xsum_sum_condsens", lib().xsum_sum_condsens(
            xp.data_ptr(), x.numel(), rule, work.data_ptr(), work.numel(), res.data_ptr(), info.data_ptr(),
            cn.data_ptr() if cn is not None else None, _stream_ptr(x.device)))
    return res, info, cn


def condsens_sum(x, rule: int = 1):
    """Host view of sum_condsens: (Result, CondSensInfo, canonical image of the truncated root)."""
    res, info, cn = sum_condsens(x, rule, canon=True)
    return (Result.from_bytes(res.cpu().numpy().tobytes()), CondSensInfo.from_bytes(info.cpu().numpy().tobytes()),
            cn.cpu().numpy().view(np.uint64).copy())


def peer_buffer_bytes(world: int) -> int:
    return int(lib().xsum_peer_buffer_bytes(world))


def peer_selftest(states, world: int, epoch: int = 1, bufs=None):
    """Run the fused multi-GPU exchange protocol with `world` virtual ranks on one GPU
    (xsum_peer_selftest): states = uint8 CUDA tensor of world state images. Returns (list of
    Result, merged images uint8 tensor [world*384], the exchange buffers for reuse)."""
    torch = _torch()
    dev = states.device
    nb = peer_buffer_bytes(world)
    if bufs is None:
        bufs = [torch.zeros(nb, dtype=torch.uint8, device=dev) for _ in range(world)]
    ptrs = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=dev)
    res = torch.zeros(world * RESULT_BYTES, dtype=torch.uint8, device=dev)
    out = torch.zeros(world * STATE_BYTES, dtype=torch.uint8, device=dev)
    _check("xsum_peer_selftest", lib().xsum_peer_selftest(states.data_ptr(), ptrs.data_ptr(), world, epoch,
                                                          res.data_ptr(), out.data_ptr(), _stream_ptr(dev)))
    rb = res.cpu().numpy().tobytes()
    return [Result.from_bytes(rb[i * RESULT_BYTES:(i + 1) * RESULT_BYTES]) for i in range(world)], out, bufs


def decode_sparse(b: bytes) -> dict:
    """Host-side parse of one sparse image (include/xsum.h): header fields and {index: digit}."""
    a = np.frombuffer(bytes(b), dtype=np.uint8)
    magic, version, w, nnz, flags, _, count = np.frombuffer(a[:24].tobytes(), dtype=np.dtype(
        [("m", "<u4"), ("v", "<u2"), ("w", "u1"), ("n", "u1"), ("f", "<u4"), ("r", "<u4"), ("c", "<u8")]))[0]
    if magic != SPARSE_MAGIC or version != VERSION or w != RADIX_BITS or a.size < 24 + 8 * int(nnz):
        raise ValueError("not a sparse xsum image")
    rec = np.frombuffer(a[24:24 + 8 * int(nnz)].tobytes(), dtype="<i8")
    digits = {int(r & 63): int(r >> 6) for r in rec}
    return {"flags": int(flags), "count": int(count), "digits": digits}


_default_acc: dict = {}
_DEFAULT_ACC_MAX = 16


def _acc_for(device) -> Accumulator:
    """The one-shot helpers' accumulator for (device, current stream): a handle is used by one
    stream at a time (include/xsum.h), so calls on different streams never share scratch/state.
    The entry holds the torch Stream object (so the stream outlives the entry) and the cache is
    LRU-bounded: an evicted entry's stream is synchronized before its buffers are released, so a
    later stream at a reused address never inherits a handle with work in flight."""
    torch = _torch()
    idx = torch.cuda.current_device() if device is None else torch.device(device).index
    key = (idx, _stream_ptr(idx))
    ent = _default_acc.pop(key, None)
    if ent is None:
        ent = (Accumulator(torch.device("cuda", idx)), torch.cuda.current_stream(idx))
        while len(_default_acc) >= _DEFAULT_ACC_MAX:
            old_key = next(iter(_default_acc))
            _, old_stream = _default_acc.pop(old_key)
            old_stream.synchronize()
    _default_acc[key] = ent                     # most recently used last
    return ent[0]


def exact_sum(x) -> tuple[Result, np.ndarray]:
    """Exact sum of a float64 / float32 / float16 / bfloat16 CUDA tensor: (rounded Result,
    canonical 34-limb image)."""
    x = _as_f64_cuda(x, allow_f32=True)
    acc = _acc_for(x.device)
    res, canon = acc.sum(x, canon=True)
    return Result.from_bytes(res.cpu().numpy().tobytes()), canon.cpu().numpy().view(np.uint64).copy()


def fsum(x) -> float:
    """Correctly rounded (RN-even) sum of a float64 CUDA tensor (float32 tensors: the correctly
    rounded binary32 of their exact sum, returned as a Python float; float16 / bfloat16
    tensors: the correctly rounded binary64 of their exact sum)."""
    x = _as_f64_cuda(x, allow_f32=True)
    res, _ = _acc_for(x.device).sum(x)
    r = Result.from_bytes(res.cpu().numpy().tobytes())
    return r.value_f32 if _is_f32(x) else r.value


_DT = {"float64": 0, "float32": 1, "float16": 2, "bfloat16": 3}


def _as_seg_input(t):
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("expected a CUDA tensor")
    if t.dtype not in (torch.float64, torch.float32, torch.float16, torch.bfloat16):
        raise TypeError(f"expected float64 / float32 / float16 / bfloat16, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t


def sum_segments(x, seg_len: int, canon: bool = False, flags: bool = False):
    """Per-segment exact sums of a CUDA tensor split into equal segments of seg_len. Values are
    the RN-even rounding of each exact sum: float64 for float64 input, float32 (the binary32
    rounding, one rounding from the exact value) for float32 / float16 / bfloat16 input.
    Returns (values[nseg], canon[nseg,34] or None, flags[nseg] or None) on the device."""
    x = _as_seg_input(x)
    if seg_len <= 0 or x.numel() % seg_len:
        raise ValueError("x.numel() must be a positive multiple of seg_len")
    return _segments(x, x.numel() // seg_len, seg_len, None, canon, flags)


def sum_segments_csr(x, offsets, canon: bool = False, flags: bool = False):
    """Variable-length segments: segment s = x[offsets[s]:offsets[s+1]] (offsets int64 CUDA)."""
    torch = _torch()
    x = _as_seg_input(x)
    if not (offsets.is_cuda and offsets.dtype == torch.int64 and offsets.is_contiguous() and offsets.numel() >= 1):
        raise TypeError("offsets must be a contiguous int64 CUDA tensor of nseg+1 entries")
    return _segments(x, offsets.numel() - 1, 0, offsets, canon, flags)


def exact_sum_dim(x, dim=-1, keepdim: bool = False):
    """Exact reduction of a CUDA tensor along one dimension: every output
    element is the correctly rounded (RN-even) sum of its fibre, independent of order - a
    reproducible torch.sum(x, dim). float64 input gives float64, float32 / float16 / bfloat16
    input the float32 rounding of the exact sum. A contiguous tensor (or a permuted view of one,
    e.g. a transpose) reduced over a non-last dimension goes to xsum_sum_strided (no copy);
    otherwise the fibres are laid out as equal contiguous segments (a movedim + contiguous copy
    for other non-contiguous inputs) and summed by
    xsum_sum_segments_ex (one warp per fibre; one lane per fibre for fibres of <= 256).
    `dim` may also be a tuple of dimensions (adjacent ones of a contiguous tensor are merged
    without a copy) or None (the exact sum of everything, a 0-d tensor, no host synchronization)."""
    torch = _torch()
    if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype not in (torch.float64, torch.float32,
                                                                           torch.float16, torch.bfloat16):
        raise TypeError("expected a float64 / float32 / float16 / bfloat16 CUDA tensor")
    f64 = x.dtype == torch.float64
    if dim is None:                              # everything: one fused sum, result stays on the device
        res, _ = _acc_for(x.device).sum(x.contiguous().reshape(-1))
        val = res[0:8].clone().view(torch.float64) if f64 else res[44:48].clone().view(torch.float32)
        out = val.reshape(())
        return out.reshape((1,) * x.dim()) if keepdim else out
    if isinstance(dim, (tuple, list)):
        if x.dim() == 0:
            raise ValueError("exact_sum_dim needs a tensor with at least one dimension")
        dims = sorted({int(k) % x.dim() for k in dim})
        if not dims:
            raise ValueError("empty dim tuple")
        if len(dims) == 1:
            return exact_sum_dim(x, dims[0], keepdim)
        red = 1
        for k in dims:
            red *= x.shape[k]
        if x.is_contiguous() and dims == list(range(dims[0], dims[-1] + 1)):
            y = x.reshape(tuple(x.shape[:dims[0]]) + (red,) + tuple(x.shape[dims[-1] + 1:]))   # a view
            out = exact_sum_dim(y, dims[0])
        else:
            keep = [k for k in range(x.dim()) if k not in dims]
            y = x.permute(keep + dims).contiguous().reshape(tuple(x.shape[k] for k in keep) + (red,))
            out = exact_sum_dim(y, -1)
        if keepdim:
            for k in dims:
                out = out.unsqueeze(k)
        return out
    if x.dim() == 0:
        raise ValueError("exact_sum_dim needs a tensor with at least one dimension")
    d = dim % x.dim()
    if not x.is_contiguous() and x.dim() > 1:
        # a permuted view of a contiguous tensor (e.g. a transpose): reduce the matching dimension
        # of the underlying contiguous layout (no copy of the input), then put the output's
        # dimensions back in the view's order
        perm = sorted(range(x.dim()), key=lambda i: -x.stride(i))
        base = x.permute(perm)
        if base.is_contiguous():
            p = perm.index(d)
            out_b = exact_sum_dim(base, p)
            rem = [perm[i] for i in range(x.dim()) if i != p]        # view dims in out_b's order
            out = out_b.permute([rem.index(k) for k in sorted(rem)]).contiguous()
            return out.unsqueeze(d) if keepdim else out
    outer = 1
    for s_ in x.shape[:d]:
        outer *= s_
    inner = 1
    for s_ in x.shape[d + 1:]:
        inner *= s_
    length = x.shape[d]
    out_shape = tuple(x.shape[:d]) + tuple(x.shape[d + 1:])
    if inner > 1 and x.is_contiguous():
        # strided fibres summed in place (xsum_sum_strided): no transposing copy
        o64, o32, _ = _strided(x, outer, length, inner, f64, not f64)
        out = (o64 if f64 else o32).reshape(out_shape)
        return out.unsqueeze(d) if keepdim else out
    xt = x.movedim(d, -1).contiguous()
    seg = xt.shape[-1]
    out_shape = xt.shape[:-1]
    nseg = 1
    for s_ in out_shape:
        nseg *= s_
    if nseg == 0:
        out = torch.empty(out_shape, dtype=torch.float64 if x.dtype == torch.float64 else torch.float32,
                          device=x.device)
    else:
        out, _, _ = _segments(xt.reshape(-1), nseg, seg, None, False, False)
        out = out.reshape(out_shape)
    return out.unsqueeze(d) if keepdim else out


def sum_strided(x, outer: int, length: int, inner: int, out64: bool = True, out32: bool = False, flags: bool = False):
    """Exact sums over the middle axis of a contiguous CUDA tensor viewed as [outer][length][inner]
    (xsum_sum_strided): returns (binary64 values or None, binary32 values or None, flags or None),
    each of outer*inner elements."""
    torch = _torch()
    if not isinstance(x, torch.Tensor) or not x.is_cuda or not x.is_contiguous() or \
            x.dtype not in (torch.float64, torch.float32, torch.float16, torch.bfloat16):
        raise TypeError("expected a contiguous float64 / float32 / float16 / bfloat16 CUDA tensor")
    if outer * length * inner != x.numel():
        raise ValueError("outer * length * inner must equal x.numel()")
    return _strided(x, outer, length, inner, out64, out32, flags)


def _strided(x, outer, length, inner, out64, out32, flags=False):
    torch = _torch()
    F = outer * inner
    o64 = torch.empty(F, dtype=torch.float64, device=x.device) if out64 else None
    o32 = torch.empty(F, dtype=torch.float32, device=x.device) if out32 else None
    fl = torch.empty(F, dtype=torch.int32, device=x.device) if flags else None
    wb = int(lib().xsum_sum_strided_work_bytes(outer, length, inner, x.device.index))
    work = torch.empty(wb, dtype=torch.uint8, device=x.device) if wb else None
    xp = x if x.numel() else torch.zeros(8, dtype=x.dtype, device=x.device)
    with torch.cuda.device(x.device):          # handle-less entry points run on the current device
        _check("xsum_sum_strided", lib().xsum_sum_strided(
            xp.data_ptr(), _DT[str(x.dtype).replace("torch.", "")], outer, length, inner,
            o64.data_ptr() if o64 is not None else None, o32.data_ptr() if o32 is not None else None,
            fl.data_ptr() if fl is not None else None, work.data_ptr() if work is not None else None, wb,
            _stream_ptr(x.device)))
    return o64, o32, fl


def _segments(x, nseg, seg_len, offsets, canon, flags):
    torch = _torch()
    f64 = x.dtype == torch.float64
    out = torch.empty(nseg, dtype=torch.float64 if f64 else torch.float32, device=x.device)
    cn = torch.empty((nseg, CANON_LIMBS), dtype=torch.int64, device=x.device) if canon else None
    fl = torch.empty(nseg, dtype=torch.int32, device=x.device) if flags else None
    xp = x if x.numel() else torch.zeros(8, dtype=x.dtype, device=x.device)
    # ragged segments: a zeroed ticket word (stream-ordered, torch's allocator) lets the
    # warps balance the work dynamically (xsum_sum_segments_ws)
    tk = torch.zeros(1, dtype=torch.int64, device=x.device) if offsets is not None else None
    with torch.cuda.device(x.device):          # handle-less entry points run on the current device
        if offsets is not None and x.numel() <= SEG_LANES_MAX * nseg:
            # mostly short CSR segments (mean length <= 256): one lane per short segment
            rc = lib().xsum_sum_segments_csr_lanes(
                xp.data_ptr(), _DT[str(x.dtype).replace("torch.", "")], nseg, offsets.data_ptr(),
                out.data_ptr() if f64 else None, None if f64 else out.data_ptr(),
                cn.data_ptr() if cn is not None else None, fl.data_ptr() if fl is not None else None,
                tk.data_ptr(), _stream_ptr(x.device))
            _check("xsum_sum_segments_csr_lanes", rc)
            return out, cn, fl
        rc = lib().xsum_sum_segments_ws(xp.data_ptr(), _DT[str(x.dtype).replace("torch.", "")], nseg, seg_len,
                                        offsets.data_ptr() if offsets is not None else None,
                                        out.data_ptr() if f64 else None, None if f64 else out.data_ptr(),
                                        cn.data_ptr() if cn is not None else None,
                                        fl.data_ptr() if fl is not None else None,
                                        tk.data_ptr() if tk is not None else None, _stream_ptr(x.device))
    _check("xsum_sum_segments_ws", rc)
    return out, cn, fl
