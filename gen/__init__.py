"""Seeded synthetic input generators shared by the oracle side (tests) and
the CUDA side (tests, bench.py).

This module holds NONE of the method's arithmetic (no PCSR, no SpMM, no
features): it only draws graphs shaped like the paper's workloads (power-law
and Poisson-like degree distributions, shuffled vs locality-ordered IDs;
P:25-27) and dense U[-1,1) matrices, as canonical CSR.  The
recipes and seeds are stated in DESIGN.md §4 ("input recipe").
"""
from .graphs import (Graph, CONFIGS, config_graph, config_B, dense, values, csr_from_pairs,  # noqa: F401
                     uniform, powerlaw, banded, community, chung_lu, roadnet_like,
                     block_lognormal, with_empty_rows, giant_row, permute)
