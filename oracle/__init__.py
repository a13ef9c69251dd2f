"""fp64 CPU oracle for the Genred hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` legs
may import this package.  The product path (paper_2004_11127_b200) never does.
"""
from .oracle import (  # noqa: F401
    build, lib_path, num_threads, set_num_threads,
    gauss_sum, gauss_gradx, lse, argkmin, sqdist_sum, softmax_grad,
)
