"""paper_2405_14009_b200 — B200-native hot path of SlipStream (arXiv 2405.14009).

The computation lives in ``libslip.so`` (CUDA for sm_100a + NCCL, C ABI in
``include/slip.h``).  This package holds the thin ctypes binding
(``_binding``) and :mod:`runtime`, which allocates device memory with torch and
passes raw pointers and streams to the library (marshalling only).
"""
from ._binding import (SLIP_AR, SLIP_B, SLIP_BC, SLIP_F, SLIP_OPT, SLIP_W, SlipError, call, lib, slip_adam,
                       slip_cluster, slip_costs, slip_io, slip_model, slip_op, slip_plan_opts, slip_report)

__all__ = ["SLIP_AR", "SLIP_B", "SLIP_BC", "SLIP_F", "SLIP_OPT", "SLIP_W", "SlipError", "call", "lib",
           "slip_adam", "slip_cluster", "slip_costs", "slip_io", "slip_model", "slip_op", "slip_plan_opts",
           "slip_report"]
