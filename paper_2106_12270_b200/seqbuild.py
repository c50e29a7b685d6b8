"""Sequential construction entry point (mirror of aliaskit/seqbuild.py).

On the device the sequential Vose order is produced by the fused pipeline:
its rows are defined by the same light/heavy merge the sequential loop
performs (seqbuild.py:33-58), evaluated from exact prefix sums instead of one
long f64 residual chain ("Formulation").  The reference's own
sequential kernel remains the correctness oracle (oracle/).
"""

from __future__ import annotations

from .model import AliasTable, WeightSet
from .pack import build_table


def vose_construct(w: WeightSet) -> AliasTable:
    """Build the alias table in Vose order (seqbuild.py:64-70)."""
    return build_table(w)
