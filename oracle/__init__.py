"""fp64 CPU oracle for the batched compressed-LoRA apply (arxiv 2407.00066).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg may import or execute anything in this package.  The product path
(paper_2407_00066_b200) never imports it and shares no code with it: no kernels, helpers,
tables or constants.  Inputs come from the neutral `workloads` package (no method arithmetic).

Every function cites the passage of PAPER.md ("P:L<n>") it follows.  Pins that tie each part to
something other than itself live in tests/test_oracle_*.py.

Parity status
  segment_ref, apply_ref, apply_dense_ref, apply_lora_ref  pinned (brute force, Prop. 1, invariants)
  project_ref                                               pinned (brute-force loops; W0 = 0 / Sigma = 0 cases)
  jd_full, sigma_star, jd_objective                         pinned (closed forms, Thm 1, Eckart-Young)
  jd_eigen_iteration, orthogonalize (App A.2)               pinned (fixed point at the App A.1 optimum,
                                                            n = 1 -> SVD subspaces, exact span, QR)
  bank_params, usage_ratio, para_saved                      pinned (App F / Table H printed values)
  random-LoRA reconstruction values (App H)   parity unpinned (distribution unknown)
"""
from .apply import segment_ref, apply_ref, apply_dense_ref, apply_lora_ref, project_ref  # noqa: F401
from .jd import (  # noqa: F401
    lora_product,
    sigma_star,
    jd_full,
    jd_full_clustered,
    jd_objective,
    mean_relative_error,
    svd_truncate,
    orthogonalize,
    jd_eigen_iteration,
)
from .accounting import bank_params, baseline_params, usage_ratio, para_saved  # noqa: F401
