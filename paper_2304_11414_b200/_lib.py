"""ctypes binding of the C-ABI library ``lib/libppmoe.so`` (include/ppmoe_capi.h).

The product path has no fallback: if the shared library is missing or fails to
load, every entry point raises.  Build it with ``make -j`` (or
``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libppmoe.so"

_P = ctypes.c_void_p
_I = ctypes.c_int
_F = ctypes.c_float
_D = ctypes.c_double
_S = ctypes.c_size_t
_U = ctypes.c_ulonglong
_UI = ctypes.c_uint
_LL = ctypes.c_longlong

# name -> (restype, argtypes); mirrors include/ppmoe_capi.h
_SIGNATURES = {
    "ppmoe_version": (_I, []),
    "ppmoe_last_error": (ctypes.c_char_p, []),
    "ppmoe_num_sms": (_I, []),
    "ppmoe_kernel_launches": (ctypes.c_ulonglong, []),
    "ppmoe_set_gemm_sm_budget": (_I, [_I]),
    "ppmoe_set_gemm_mode": (_I, [_I]),
    "ppmoe_set_gemm_narrow": (_I, [_I]),
    "ppmoe_route_workspace_bytes": (_S, [_I, _I, _I]),
    "ppmoe_route_workspace_bytes_h": (_S, [_I, _I, _I, _I]),
    "ppmoe_route": (_I, [_P, _I, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _S, _P]),
    "ppmoe_route_combine_stats": (_I, [_P, _I, _I, _I, _P, _P, _P]),
    "ppmoe_dispatch_workspace_bytes": (_S, [_I, _I, _I]),
    "ppmoe_dispatch_plan": (_I, [_P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _I, _P, _S, _P]),
    "ppmoe_a2a_compact": (_I, [_P, _P, _P, _P, _I, _P, _P, _I, _P, _P, _P, _P, _P]),
    "ppmoe_a2a_owner_layout": (_I, [_P, _I, _I, _I, _P, _P, _P]),
    "ppmoe_scatter_rows": (_I, [_P, _I, _I, _P, _P, _P, _P, _P]),
    "ppmoe_a2a_permute_rows": (_I, [_P, _I, _I, _I, _P, _P, _P]),
    "ppmoe_gather": (_I, [_P, _I, _I, _I, _P, _I, _P, _P, _I, _P, _P, _P, _P]),
    "ppmoe_chunk_rows": (_I, [_P, _P, _P, _I, _I, _I, _P, _P, _P]),
    "ppmoe_expert_fc1_fwd": (_I, [_I, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P]),
    "ppmoe_expert_fc2_fwd": (_I, [_I, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _I, _F, _P, _P, _P, _P, _P]),
    "ppmoe_combine": (_I, [_I, _P, _P, _I, _P, _P, _I, _I, _I, _P, _P, _I, _P, _P]),
    "ppmoe_input_grads_workspace_bytes": (_S, [_I, _I, _I, _I]),
    "ppmoe_input_grads": (_I, [_I, _P, _P, _I, _P, _I, _I, _I, _P, _P, _P, _I, _P, _P, _P, _S, _P]),
    "ppmoe_cast_out": (_I, [_P, _I, _P, _I, _P]),
    "ppmoe_ipc_handle_bytes": (_S, []),
    "ppmoe_ipc_alloc": (_I, [_S, _P, _P]),
    "ppmoe_ipc_open": (_I, [_P, _P]),
    "ppmoe_ipc_close": (_I, [_P]),
    "ppmoe_ipc_free": (_I, [_P]),
    "ppmoe_nvl_pad_bytes": (_S, []),
    "ppmoe_nvl_barrier": (_I, [_P, _I, _I, _I, _UI, _P, _LL, _P]),
    "ppmoe_nvl_owner_gather": (_I, [_P, _P, _I, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _I, _P, _P, _P, _I, _P]),
    "ppmoe_nvl_pull_blocks": (_I, [_P, _I, _I, _I, _I, _P, _P]),
    "ppmoe_nvl_sum_rows": (_I, [_P, _I, _I, _I, _I, _P, _P]),
    "ppmoe_nvl_sum_all": (_I, [_P, _I, _I, _P, _P]),
    "ppmoe_nvl_route_gather": (_I, [_P, _I, _I, _I, _I, _P, _P, _P, _P, _P]),
    "ppmoe_nvl_pull_blocks_ce": (_I, [_P, _I, _I, _I, _I, _P, _P]),
    "ppmoe_nvl_pull_range_ce": (_I, [_P, _I, _I, _I, _I, _I, _I, _P, _P]),
    "ppmoe_expert_fc2_fwd_owner": (_I, [_I, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P, _I, _F, _P, _P, _P, _P, _P, _I, _I,
                                        _P]),
    "ppmoe_nvl_sum_slots": (_I, [_P, _I, _I, _I, _I, _P, _P, _P, _P]),
    "ppmoe_nvl_cast_owned": (_I, [_P, _I, _I, _P, _P, _P]),
    "ppmoe_bwd_dy": (_I, [_I, _P, _P, _P, _I, _I, _I, _P, _P, _I, _F, _P, _P, _P, _P, _P]),
    "ppmoe_dropout_stream": (_I, [_P, _I, _I, _I, _I, _U, _U, _U, _U, _P, _P]),
    "ppmoe_expert_fc2_dgrad": (_I, [_I, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P, _P]),
    "ppmoe_expert_fc2_wgrad": (_I, [_I, _P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _P]),
    "ppmoe_expert_fc1_dgrad": (_I, [_I, _P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _P]),
    "ppmoe_expert_fc1_wgrad": (_I, [_I, _P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _P]),
    "ppmoe_gate_bwd": (_I, [_P, _P, _P, _P, _P, _I, _P, _I, _I, _I, _P, _P, _P]),
    "ppmoe_gate_grad_workspace_bytes": (_S, [_I, _I, _I]),
    "ppmoe_gate_grads": (_I, [_P, _P, _I, _P, _P, _I, _I, _I, _P, _P, _P, _S, _P]),
    "ppmoe_gemm_selftest": (_I, [_I, _I, _I, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P]),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lib = None


class PPMoEError(RuntimeError):
    """A CUDA-side failure reported by the C-ABI (negative status -2/-4)."""


def load():
    """Load (once) and return the ctypes handle; raise loudly if unavailable."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"PPMoE CUDA library not built: {LIB_PATH} is missing (run `make -j` in the repo root). "
                "There is no CPU fallback for the product path."
            )
        lib = ctypes.CDLL(os.fspath(LIB_PATH))
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


_FNS: dict = {}
_FAST = None  # the CPython fast-call bindings (lib/_fastcall*.so), loaded with the library


def _load_fast():
    """The generated CPython bindings of the same C-ABI (csrc/fastcall.c, built next to
    libppmoe.so): ~1 us per call instead of ctypes' ~14 us.  Absent (e.g. a build without
    Python headers) -> the ctypes binding of the same library is used."""
    global _FAST
    if _FAST is None:
        import importlib.machinery
        import importlib.util
        import sysconfig

        load()  # the library itself must be present: no fallback for it
        path = LIB_PATH.parent / ("_fastcall" + sysconfig.get_config_var("EXT_SUFFIX"))
        mod = False
        if path.exists() and os.environ.get("PPMOE_CTYPES") != "1":
            loader = importlib.machinery.ExtensionFileLoader("_fastcall", os.fspath(path))
            spec = importlib.util.spec_from_file_location("_fastcall", os.fspath(path), loader=loader)
            mod = importlib.util.module_from_spec(spec)
            loader.exec_module(mod)
        _FAST = mod
    return _FAST


def query(name: str, *args):
    """A value-returning C-ABI function (workspace sizes, counts): no status translation."""
    fn = _FNS.get(name)
    if fn is None:
        fast = _load_fast()
        fn = _FNS[name] = (getattr(fast, name, None) if fast else None) or getattr(load(), name)
    return fn(*args)


def call(name: str, *args) -> int:
    """Invoke one C-ABI entry point and translate its status to an exception."""
    fn = _FNS.get(name)
    if fn is None:
        fast = _load_fast()
        fn = _FNS[name] = (getattr(fast, name, None) if fast else None) or getattr(load(), name)
    rc = fn(*args)
    if rc != 0:
        lib = load()
        msg = lib.ppmoe_last_error().decode(errors="replace")
        if rc in (-1, -3):
            raise ValueError(msg)
        raise PPMoEError(f"{name}: {msg} (status {rc})")
    return rc


def ptr(t: torch.Tensor | None):
    """Raw device pointer of a tensor as an int (ctypes passes it as void*; None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(device=None):
    """The current CUDA stream of `device` (default: the current device) as a raw handle.
    Uses torch's raw-stream query: no torch.cuda.Stream object per C-ABI call (that object
    construction was ~20 us, a fifth of the host enqueue time of a layer step)."""
    idx = torch._C._cuda_getDevice() if device is None else torch.cuda._utils._get_device_index(device)
    return torch._C._cuda_getCurrentRawStream(idx)
