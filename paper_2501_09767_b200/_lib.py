"""ctypes binding of liblemo.so (the C ABI in include/lemo.h).

The library is built in-tree (``paper_2501_09767_b200/liblemo.so``).  There is
no fallback: if the library is missing or a call fails, an exception is
raised.  Argument types are derived from the declarations in
``include/lemo.h`` itself, so the binding cannot drift from the header.
Pointers are passed as integers (``tensor.data_ptr()``), streams as the raw
``cudaStream_t`` of torch's current stream.
"""

from __future__ import annotations

import ctypes
import os
import re
from pathlib import Path

import torch

_PKG = Path(__file__).resolve().parent
# LEMO_LIB overrides the library path (A/B builds of the same sources)
_LIB_PATH = Path(os.environ["LEMO_LIB"]) if os.environ.get("LEMO_LIB") else _PKG / "liblemo.so"
HEADER = _PKG.parent / "include" / "lemo.h"

_CT = {"p": ctypes.c_void_p, "i": ctypes.c_int, "f": ctypes.c_float, "d": ctypes.c_double,
       "l": ctypes.c_longlong}
_RET = {"int": ctypes.c_int, "void": None, "const char*": ctypes.c_char_p, "double": ctypes.c_double}


class LemoError(RuntimeError):
    pass


def _param_code(decl: str) -> str:
    decl = decl.strip()
    if "*" in decl:
        return "p"
    base = decl.rsplit(None, 1)[0] if " " in decl else decl
    base = base.replace("const", "").strip()
    if base in ("int", "int32_t"):
        return "i"
    if base == "float":
        return "f"
    if base == "double":
        return "d"
    if base in ("long long", "int64_t"):
        return "l"
    raise ValueError(f"unsupported parameter type in lemo.h: {decl!r}")


def parse_header(path: Path = HEADER) -> dict[str, tuple[str, str]]:
    """name -> (return type, parameter codes) for every lemo_* declaration."""
    text = re.sub(r"/\*.*?\*/", "", path.read_text(), flags=re.S)
    text = re.sub(r"//[^\n]*", "", text)
    out: dict[str, tuple[str, str]] = {}
    for m in re.finditer(r"(int|void|const char\*|double)\s+(lemo_\w+)\s*\(([^)]*)\)\s*;", text):
        ret, name, params = m.group(1), m.group(2), m.group(3).strip()
        if params in ("", "void"):
            codes = ""
        else:
            codes = "".join(_param_code(p) for p in params.split(","))
        out[name] = (ret, codes)
    return out


SIGNATURES = parse_header()
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise LemoError(
                f"{_LIB_PATH} is missing: build it with `python -m paper_2501_09767_b200.build` "
                "(there is no CPU fallback)")
        handle = ctypes.CDLL(str(_LIB_PATH))
        for name, (ret, codes) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.argtypes = [_CT[c] for c in codes]
            fn.restype = _RET[ret]
        _lib = handle
    return _lib


def memory_allocated(device) -> int:
    """torch.cuda.memory_allocated without flattening the whole statistics
    dict in Python (that costs ~0.2 ms, and the step reads it twice)."""
    idx = device.index if isinstance(device, torch.device) and device.index is not None \
        else torch.cuda.current_device()
    try:
        return int(torch._C._cuda_memoryStats(idx)["allocated_bytes"]["all"]["current"])
    except (AttributeError, KeyError, TypeError):  # pragma: no cover - other torch builds
        return torch.cuda.memory_allocated(idx)


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    """Raw cudaStream_t of `stream` (default: torch's current stream on the
    current device) — the cheap C query, this runs once per launch."""
    if stream is not None:
        return int(stream.cuda_stream)
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


def ptr(t) -> int | None:
    """Device address of a tensor (None for None)."""
    return None if t is None else t.data_ptr()


# kernels launched per entry point (everything else launches exactly one)
_LAUNCHES = {"lemo_flash_bwd_tc": 3, "lemo_lora_grads": 2}


class Instrument:
    """Launch counting and per-entry-point CUDA-event timing (bench.py).

    counting: launches[name] += kernels launched by each call.
    timing:   for names in `timed`, a (start, end) event pair is recorded on
              the current stream around every call.
    """

    def __init__(self):
        self.enabled = False
        self.launches: dict[str, int] = {}
        self.timed: set[str] = set()
        self.events: dict[str, list] = {}
        self.notes: dict[str, list] = {}

    def reset(self, timed=()):
        self.launches = {}
        self.timed = set(timed)
        self.events = {n: [] for n in self.timed}
        self.notes = {n: [] for n in self.timed}

    def note(self, name: str, value) -> None:
        """Per-call metadata (e.g. the row count) for timed entry points."""
        if self.enabled and name in self.notes:
            self.notes[name].append(value)

    def total_launches(self) -> int:
        return sum(self.launches.values())

    def elapsed_ms(self, name: str) -> list[float]:
        return [a.elapsed_time(b) for a, b in self.events.get(name, [])]


INSTRUMENT = Instrument()


_FNS: dict = {}


def call(name: str, *args):
    """Invoke a status-returning entry point; raise LemoError on failure."""
    fn = _FNS.get(name)
    if fn is None:
        fn = _FNS[name] = getattr(lib(), name)
    ins = INSTRUMENT
    if ins.enabled:
        ins.launches[name] = ins.launches.get(name, 0) + _LAUNCHES.get(name, 1)
        if name in ins.timed:
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            rc = fn(*args)
            b.record()
            ins.events[name].append((a, b))
        else:
            rc = fn(*args)
    else:
        rc = fn(*args)
    if rc != 0:
        msg = lib().lemo_last_error().decode(errors="replace")
        raise LemoError(f"{name} failed ({rc}): {msg}")
    return rc
