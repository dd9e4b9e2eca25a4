"""Seeded synthetic inputs for shared-prefix decode attention.

This module is the ONLY code shared between the oracle tests (`oracle/`) and the
CUDA path (`paper_2402_05099_b200/`).  It draws random numbers and lays them out;
it contains none of the method's arithmetic (no scores, softmax, LSE or combine).
"""
from .gen import (  # noqa: F401
    PagedCache,
    Problem,
    TreeProblem,
    bf16_bits_to_f32,
    f32_to_bf16_bits,
    make_problem,
    make_tree_problem,
    normal_f32,
    normal_bf16_bits,
    paginate,
    BF16_NAN,
    two_level_tree,
)
