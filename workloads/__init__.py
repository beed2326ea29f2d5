"""Seeded synthetic workloads shared by the oracle and the CUDA path.

This package holds *data only*: model graph descriptors (the tenants' DFGs
M_n = [O_{n,1}..O_{n,i}], §4.1 l.605-607) and seeded tensor
generators.  It contains none of the method's
arithmetic: no convolution, no normalisation, no scheduling.  Both
``oracle/`` and ``paper_2304_11745_b200/`` consume what it produces; neither
is imported here.
"""
from .zoo import (  # noqa: F401
    Graph, MODELS, build_model, CONFIGS, config_tenants,
)
from .gen import (  # noqa: F401
    bf16_round, make_params, make_input, make_labels, tenant_seed,
)
