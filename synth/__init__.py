"""Seeded synthetic inputs shared by the oracle, the tests and the bench.

This package holds NO arithmetic of the method (no filter, no projection, no
interval estimate): it only builds the sparse symmetric matrices ``A`` (CSR)
and the Gaussian starting blocks ``X0`` of the five BASELINE.json configs and
of small analogues, exactly as DESIGN.md's input recipe states (SURVEY.md
§8c-11..15, §8d).  Both the CPU oracle (``oracle/``) and the CUDA path
(``paper_1507_06078_b200``) consume what it returns; neither is imported here.
"""
from .generators import (  # noqa: F401
    CSR,
    laplacian_1d,
    laplacian_2d,
    laplacian_3d_potential,
    stencil27_3d,
    zipf_random,
    diagonal,
    gaussian_block,
    gaussian_block_rows,
)
from .configs import CONFIGS, SMALL_ANALOGS, build_config, starting_block, ConfigSpec  # noqa: F401
