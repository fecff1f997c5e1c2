"""Import-path alias of the reference's ``paco.matmul`` (semiring MM API)."""

from .cuboid import (DEFAULT_BASE, Cuboid, longest_axis, mm_hetero_partition, mm_one_piece_partition,
                     mm_paco_partition, temp_shape)
from .mm import measured_weights, mm_execute, mm_oracle, mm_seq
from .semiring import (ALL_SEMIRINGS, MINPLUS_INF, SEMIRING_BF16, SEMIRING_F32, SEMIRING_F32_SIMT, SEMIRING_F64,
                       SEMIRING_INT, SEMIRING_MAXPLUS, SEMIRING_MINPLUS, SEMIRING_MINPLUS_SAT,
                       SEMIRINGS, TROPICAL_INF, Semiring)

__all__ = ["DEFAULT_BASE", "Cuboid", "longest_axis", "mm_hetero_partition", "mm_one_piece_partition",
           "mm_paco_partition", "temp_shape", "measured_weights", "mm_execute", "mm_oracle", "mm_seq", "ALL_SEMIRINGS",
           "MINPLUS_INF", "SEMIRING_BF16", "SEMIRING_F32", "SEMIRING_F32_SIMT", "SEMIRING_F64", "SEMIRING_INT",
           "SEMIRING_MAXPLUS", "SEMIRING_MINPLUS", "SEMIRING_MINPLUS_SAT", "SEMIRINGS",
           "TROPICAL_INF", "Semiring"]
