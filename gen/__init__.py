"""Seeded synthetic inputs for the sFLSQR/sFLSMR hot path (BASELINE.json configs).

INPUT INFRASTRUCTURE ONLY: shared by the CPU oracle (``oracle/``) and the CUDA
path (``paper_2605_22281_b200``).  It builds A (and B), x_true, noise and b; it
holds none of the method's arithmetic.  See DESIGN.md "Input recipe".
"""
from .problems import (  # noqa: F401
    CSR,
    Problem,
    SolverSpec,
    build_lib,
    make_problem,
    siddon_csr,
    pixbp_csr,
    ellipse_phantom,
    CONFIGS,
)
