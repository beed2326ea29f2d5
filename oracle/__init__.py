"""GACER parity oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2304_11745_b200``) never imports it, and it imports
nothing from the product path: the two share no code.  Inputs come from the
data-only ``workloads`` package.

Contents
--------
* ``ops``      -- ctypes binding of ``gacer_oracle.c`` (plain fp64 operators).
* ``forward``  -- y_n = M_n(x_n): op-by-op fp64 interpretation of a tenant DFG
                  (§4.1 l.605-607; semantics SURVEY §8(c) C1), and
                  ``chunked_forward``: Eq. 5 applied literally (split, compute,
                  concat; §4.2 l.657-675).
* ``train``    -- the training tenant (A11): BN-train forward, plain
                  backward operators (``gacer_oracle_train.c``), mean
                  softmax-CE, SGD momentum, and the replicas' gradient mean
                  (A12, ``allreduce_mean``).  Pinned by finite differences,
                  closed forms and PyTorch fp64 autograd (test_oracle_train.py).
* ``plan``     -- the paper's plan semantics: segmentation by pointers (Eq. 7,
                  l.742-753) and clusters (Eq. 6, l.723-739).

Parity pins (tests/test_oracle_*.py): hand-computed convolution, closed forms
for constant inputs, torch-CPU fp64 library routines for every operator and
whole tenants, batch independence, Eq. 5 decomposition invariance, the Eq. 6/7
worked examples of the paper (tests/golden/).
"""
from . import ops, forward, plan, train  # noqa: F401
from .forward import forward_graph, chunked_forward  # noqa: F401
