"""fp64 CPU oracle of the implicit-SVD hot path (arXiv 2111.06312).

TEST INFRASTRUCTURE ONLY.  Nothing on the product path may import this
package: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` leg / ``--impl reference`` arm call it.  It shares no code
with ``paper_2111_06312_b200`` (no kernels, headers, helpers, constants or
pre/post-processing); both sides only read the seeded inputs of ``synth/``.

Every function cites the PAPER.md passage it follows (``P:n`` = line n of
/root/reference/PAPER.md).  Parity pins live in ``tests/test_oracle_*.py``
and ``tests/golden/``.  Parity status per function is listed in DESIGN.md
("Oracle pins"); no function here is "parity unpinned".
"""
from .isvd_oracle import (  # noqa: F401
    NCOperator,
    NEOperator,
    RowSubsetOperator,
    adjacency,
    context_weights,
    embeddings,
    exact_svd,
    isvd,
    label_reuse_adj,
    least_norm,
    orthonorm_cholesky,
    orthonorm_qr,
    pinv_diag,
    sign_fix,
    spectral_kernel,
    sym_norm_adj,
    transition,
    uniform_weights,
)
from .philox import omega as philox_omega, philox4x32_10  # noqa: F401
