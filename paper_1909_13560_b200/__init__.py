"""B200-native multistep BSDE solver (Kapllani & Teng, arXiv 1909.13560).

The product path is the CUDA library ``libbsde_b200.so`` behind the C ABI in
``include/bsde.h``; ``bsde`` is its thin ctypes binding.  ``workloads`` holds the
problem parameters of the paper's examples and BASELINE.json's configs.
"""
from . import workloads  # noqa: F401
from .bsde import (  # noqa: F401
    BsdeError, Solver, GroupSolver, bsde_config, bsde_result, load_library, make_config, query_workspace,
    query_partition, nccl_unique_id, solve_batch, measure_fp64_peak, EXPORTS,
)
