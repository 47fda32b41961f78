"""Oracle for the parameter accounting of App F and the "Para. Saved" column of Table H.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

App F:
  baseline     D * 2 * 16
  JD-Full      D * 2 * r + N * r^2
  clustering   D * 2 * r * c + N * (r^2 + 1)      ("+1" = the cluster assignment)
with D = 4096 (the printed "4098", is read as 4096: SURVEY 8(c) c5 #5).
Table H "Para. Saved" is two-valued "per-adapter / total" (decoding SURVEY 8(c) c5 #7):
  per-adapter  1 - |Sigma_i| / (2 D 16)
  total        1 - (shared + N |Sigma_i|) / (N 2 D 16)
with |Sigma_i| = r^2 (full), r (diag), r^2 + 1 (clustered) and, for the per-LoRA SVD of Eq. 4,
|Sigma_i| = 2 D r with nothing shared.
"""

D_MISTRAL = 4096
BASE_RANK = 16


def baseline_params(D: int = D_MISTRAL) -> int:
    return D * 2 * BASE_RANK


def _per_adapter(method: str, r: int, D: int) -> int:
    return {"full": r * r, "diag": r, "clus": r * r + 1, "svd": 2 * D * r}[method]


def _shared(method: str, r: int, clusters: int, D: int) -> int:
    return {"full": 2 * D * r, "diag": 2 * D * r, "clus": 2 * D * r * clusters, "svd": 0}[method]


def bank_params(method: str, N: int, r: int, clusters: int = 1, D: int = D_MISTRAL) -> int:
    """Params_JD_Full / Params_Clustering for one module."""
    return _shared(method, r, clusters, D) + N * _per_adapter(method, r, D)


def usage_ratio(method: str, N: int, r: int, clusters: int = 1, D: int = D_MISTRAL) -> float:
    """GPU Usage Ratio = Params / Params_baseline."""
    return bank_params(method, N, r, clusters, D) / baseline_params(D)


def para_saved(method: str, N: int, r: int, clusters: int = 1, D: int = D_MISTRAL):
    """(per-adapter, total) parameter-saved ratios of Table H."""
    base = baseline_params(D)
    per = 1.0 - _per_adapter(method, r, D) / base
    total = 1.0 - bank_params(method, N, r, clusters, D) / (N * base)
    return per, total
