"""B200-native expert-parallel dispatch/combine (arXiv 2512.19849 / UCCL-EP path).

Public surface:
* ``Buffer``, ``Config``, ``EventOverlap`` — DeepEP-compatible API
* ``LocalGroup`` — R ranks on one GPU (single-GPU multi-rank test harness)
* ``command``, ``imm``, ``kernels``, ``fifo`` — drop-ins for the reference's
  epsim.command / epsim.imm / epsim.kernels and the FifoChannel of SPEC.md:17-124
* ``per_token_cast_to_fp8`` — the LL FP8 quantiser as a standalone op

Everything executes in libepb200.so (csrc/); importing fails loudly if the
library has not been built.
"""
import os as _os

# The CPU proxy issues copies on its own streams while kernels spin on their
# completion; CUDA multiplexes streams onto CUDA_DEVICE_MAX_CONNECTIONS hardware
# queues (default 8), and a copy sharing a queue with such a kernel would wait
# behind it.  More queues make that sharing unlikely; this only takes effect
# if the package is imported before the process creates its CUDA context.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from . import _lib  # noqa: F401,E402  (loads libepb200.so or raises)
from .buffer import Buffer, Config, EventOverlap, LocalGroup, nvl_bytes_hint, ring_nvl_bytes
from .errors import (ChannelShutdown, ConfigError, ConnectionError_, EpsimError, FaultError, InvariantViolation,
                     ProtocolViolation, RingDeadlock, UnsupportedOperation)
from .ops import per_token_cast_to_fp8

__all__ = ["Buffer", "Config", "EventOverlap", "LocalGroup", "nvl_bytes_hint", "ring_nvl_bytes", "per_token_cast_to_fp8",
           "EpsimError", "ProtocolViolation", "ChannelShutdown", "ConfigError", "FaultError", "ConnectionError_",
           "UnsupportedOperation", "InvariantViolation", "RingDeadlock"]
