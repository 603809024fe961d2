"""B200-native particle-window cost engine for SIRD calibration (arXiv 2204.12346).

The hot path — every PSO particle integrating the SIRD model with explicit
Euler over a calibration window and scoring it against the observed series
(reference: /root/reference/proj/src/calibration.cpp:120-155, model.cpp:76-107,
objectives.cpp:95-120) — runs as hand-written sm_100a CUDA kernels behind the
C-ABI in include/sirdgpu.h.  This package is the Python side of that
boundary; there is no CPU fallback.
"""
from . import errors
from ._capi import Context, Plan, Window, parse_spec, probe_fp64_rate

__all__ = ["Context", "Plan", "Window", "errors", "parse_spec", "probe_fp64_rate"]
