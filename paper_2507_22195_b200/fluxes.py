"""Interface-flux family selector (reference fluxes.py:26-43).

The flux algebra itself runs on the device (csrc/mhdg_math.cuh); this module
keeps the reference's configuration object and its validation.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import InvalidConfig

FLUX_KINDS = ("lf", "ec", "es", "kepes")
FLUX_CODE = {"lf": 0, "ec": 1, "es": 2, "kepes": 3}


@dataclass(frozen=True)
class DissipationSpec:
    """lf: central + scalar wavespeed dissipation; ec: entropy conservative;
    es: ec + scalar dissipation on the state jump; kepes: ec + eigenvector
    scaled dissipation on the entropy-variable jump."""

    kind: str = "kepes"

    def __post_init__(self):
        if self.kind not in FLUX_KINDS:
            raise InvalidConfig(f"flux kind {self.kind!r} not one of {FLUX_KINDS}")

    @property
    def code(self):
        return FLUX_CODE[self.kind]
