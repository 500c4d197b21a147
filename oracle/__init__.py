"""fp64 CPU oracle for the SlipStream decoupled-B/W stage step — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import anything in this package.  The product
path (``paper_2405_14009_b200``) never imports it and shares no code with it:
no kernels, headers, helpers, constant tables or pre/post-processing.  The only
shared module is ``slipdata`` (seeded input generators, no method arithmetic).

Modules
  layer.py     one pre-LN GPT layer: forward, coupled backward, B (input
               grads) / W (weight grads) split            (§3.2)
  adam.py      AdamW with bias correction                 (§4.3, "AdamW")
  pipeline.py  DP x PP numerics with re-routing, canonical-order gradient sum,
               per-worker accumulation in plan order      (§3.1, §3.4)
  planner.py   recoverability, round-robin assignment, 1F1B / decoupled /
               staggered list scheduler, validator (Eqs. 2-6)
                                                          (§3.1-3.4, §4.2)

Pins (what ties each function to something other than itself) are listed in
DESIGN.md "Oracle pins" and exercised by ``tests/test_oracle_*.py``.
Parity unpinned: heuristic schedules beyond the pinned paper cases are only
constrained by the validator and lower bounds (DESIGN.md "Readings" R17, R22).
"""
