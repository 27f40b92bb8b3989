"""Configuration and run-info types (drop-in for helmfmm's dataclasses).

FmmConfig/MacParams/FmmInfo/InteractionEvent keep the fields, defaults and
validation of traversal.py:46-85; TreeConfig those of tree.py:36-45.  The
extra FmmConfig field ``dtype`` selects the device storage precision: "c128"
(the reference's complex128, kernel.py:68, tree.py:147; all arithmetic FP64)
or "c64" (complex64 storage and streams: coordinate differences are formed in
FP64 and rounded once; P2M/M2M/L2L, M2F, the Hadamard M2L products and per-row
sums and the P2P pair terms and sums run in FP32; the F2L, the L2P sum and the
near + far combine run in FP64 -- include/defmm_b200.h).
"""

from __future__ import annotations

from dataclasses import dataclass, field

STRATEGIES = ("t", "t+s", "t+s+r")  # interpolation.py:36
DTYPES = ("c128", "c64")


@dataclass(frozen=True)
class TreeConfig:
    ncrit: int = 64
    hard_depth_cap: int = 30

    def __post_init__(self):
        if self.ncrit < 1:
            raise ValueError("ncrit must be >= 1")
        if self.hard_depth_cap < 0:
            raise ValueError("hard_depth_cap must be >= 0")


@dataclass(frozen=True)
class FmmConfig:
    order: int = 5
    ncrit: int = 64
    eta: float = 1.0
    kappa: float = 0.0
    # the three reference strategies agree to 1e-13 (test_interpolation.py:194-204)
    # and all map to the same fused device kernels; the field is kept and validated
    strategy: str = "t+s+r"
    hf_switch: float = 2.0
    hard_depth_cap: int = 30
    dtype: str = "c128"

    def __post_init__(self):
        if self.order < 2:
            raise ValueError("order must be >= 2")
        if self.order > 8:
            # boundary deviation: the reference accepts any order
            # >= 2 (traversal.py:58-60); the device kernels are instantiated for
            # P = 2L-1 <= 15 (BASELINE's sweep stops at L = 8)
            raise ValueError("the B200 kernels are compiled for orders 2..8 (the reference accepts any order >= 2)")
        if self.strategy not in STRATEGIES:
            raise ValueError(f"strategy must be one of {STRATEGIES}")
        if not (self.eta > 0):
            raise ValueError("eta must be > 0")
        if self.kappa < 0:
            raise ValueError("kappa must be >= 0")
        if self.dtype not in DTYPES:
            raise ValueError(f"dtype must be one of {DTYPES}")


@dataclass(frozen=True)
class MacParams:
    eta: float = 1.0
    kappa: float = 0.0
    hf_threshold: float = 2.0

    def __post_init__(self):
        if not (self.eta > 0):
            raise ValueError("eta must be > 0")


@dataclass(frozen=True)
class InteractionEvent:
    kind: str  # "M2L" | "P2P"
    target: object
    source: object
    direction: object = None


@dataclass
class FmmInfo:
    timings: dict = field(default_factory=dict)
    counts: dict = field(default_factory=dict)
    hf_max_level: int = -1
