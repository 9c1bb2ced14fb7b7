"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This package holds NONE of the method's arithmetic (no supports, no currTable,
no GAC); it only draws random numbers and lays out inputs.  It is the one module
both sides of a parity check may import ("input recipe").
"""
from .rng import Rng, splitmix64  # noqa: F401
from .tables import (  # noqa: F401
    table1, random_table, banded_table, knapsack_table, LIN_PRESETS, Problem,
    short_table, negative_table, STAR,
)
from .layout import (  # noqa: F401
    member_to_bitmap, bitmap_to_member, dom_word_offsets, full_member,
)
from .policies import bulk_removal, walk_removal, fix_one_value_removal  # noqa: F401
