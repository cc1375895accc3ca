"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the method (no gate application, no
branch expansion, no reconstruction, no sampling).  It only produces inputs:

* ``circuits``  - universal random grid circuits (gate lists) under the
  Ref. [6]-style rules reconstructed in SURVEY App. A.1.
* ``blocks``    - the sampled upper/lower bitstring index blocks S_u, S_l
  (SURVEY §8(c) Q9).
* ``synthetic`` - seeded synthetic arrays (probabilities, branch slices) for
  the stand-alone sampler and branch-sum boundary tests.

Both ``oracle/`` and the product package may import it; neither imports the
other.
"""
from .circuits import (Circuit, SX, SY, T, CZ, KIND_NAMES, generate, config_circuit,
                       CONFIGS, layouts, cz_period)
from .blocks import sample_block
from . import synthetic

__all__ = ["Circuit", "SX", "SY", "T", "CZ", "KIND_NAMES", "generate", "config_circuit",
           "CONFIGS", "layouts", "cz_period", "sample_block", "synthetic"]
