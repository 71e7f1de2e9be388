"""Device plumbing: torch owns device memory and streams, the native library
does the work.  No CPU fallback exists -- without CUDA every hot-path entry
point raises."""

from __future__ import annotations

import ctypes

import torch

from ._lib import check, lib


class NoDevice(RuntimeError):
    pass


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise NoDevice("paper_2311_12133_b200 runs on a CUDA device only (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def bind() -> None:
    """Point the library's runtime at torch's current device."""
    check(lib().hpez_set_device(torch.cuda.current_device()), "hpez_set_device")


def stream() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> ctypes.c_void_p:
    if t is None:
        return ctypes.c_void_p(0)
    return ctypes.c_void_p(t.data_ptr())
