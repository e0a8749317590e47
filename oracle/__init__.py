"""ORACLE — test infrastructure, NOT part of the product path.

A plain, slow, obviously-correct CPU implementation of what the hot path computes
(§3.1 Alg. 1, Defs. 3 and 6, Alg. 2), written from the paper's text in FP64.
Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import or execute anything under `oracle/`.  It shares no
code with `paper_2311_03393_b200/` (the CUDA path) and imports nothing from it; both
sides consume inputs from `synthgen/` only.

Citation key: "P:L<a>-<b>" = /root/reference/PAPER.md lines; "S:L<a>-<b>" = SPEC.md
lines (used for the paper-gap readings, listed in DESIGN.md §3).

Pinning (see tests/test_oracle_pins.py): every function below is pinned to something
other than itself — a library routine (scipy cdist, numpy BLAS), a closed form, an
invariant, brute force on tiny inputs, or a worked value; see DESIGN.md §4 for the table.
"""
from .hashplan import splitmix64_stream, cw_params, plan_count_sketch  # noqa: F401
from .reference import (  # noqa: F401
    OracleError, stream_stats, znormalize, sketch, window_stats, znorm_windows, dist,
    selfjoin_brute, selfjoin_rows, selfjoin_tierb, combine, topk_greedy, detect, dimension_detection, refine, abjoin_brute,
)
