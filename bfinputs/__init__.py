"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

Holds factor containers, generators (random / closed-form / kernel-compressed) and
right-hand sides.  It contains no butterfly-apply arithmetic ("Inputs").
"""
from .factors import (Butterfly, HODBF, Stage, bitrev, butterfly_from_blocks, dft_butterfly,
                      identity_butterfly, random_butterfly, random_level_maps, random_ranks_butterfly,
                      random_rhs, slot_ordered, uniform_leaf_ptr)

__all__ = ["Butterfly", "HODBF", "Stage", "bitrev", "butterfly_from_blocks", "dft_butterfly",
           "identity_butterfly", "random_butterfly", "random_level_maps", "random_ranks_butterfly",
           "random_rhs", "slot_ordered", "uniform_leaf_ptr"]
