"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NONE of the method's arithmetic (no operator, no
orthonormalisation, no SVD, no Omega draw).  It only produces the graphs
(CSR), the feature matrices X and the per-config solver parameters that stand
in for the paper's datasets (Table 1), following the
recipes in SURVEY.md section 8(d) and the readings listed in DESIGN.md.

Everything is deterministic from (config seed, stream label) through a
counter-based SplitMix64 stream written out in `synth/streams.py`, so the
bytes do not depend on the numpy version.
"""
from .configs import CONFIGS, get_config, solver_params  # noqa: F401
from .graphs import Graph, make_graph, make_features, powerlaw_graph, sbm_graph, uniform_graph  # noqa: F401
