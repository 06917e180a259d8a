"""B200-native linear-time Silhouette (arXiv 2303.14102): the fastsil hot path
rebuilt as hand-written sm_100a CUDA behind a C ABI (include/fsil.h).

    from paper_2303_14102_b200 import compute_silhouette
    report = compute_silhouette(X, labels, metric="cosine")

See DESIGN.md for the kernels and INTEGRATION.md for the reference-side bindings.
"""
from .api import (  # noqa: F401
    COSINE, EUCLID, PATH_AUTO, PATH_FFMA, PATH_TCGEN05, SQEUCLID, Context, FsilError, IoError,
    SilhouetteReport, ValidationError, assemble_score, compute_silhouette, default_context, lib,
    metric_code, plan_shards,
)

__all__ = ["compute_silhouette", "Context", "SilhouetteReport", "ValidationError", "IoError",
           "FsilError", "plan_shards", "assemble_score", "SQEUCLID", "COSINE", "EUCLID",
           "PATH_AUTO", "PATH_FFMA", "PATH_TCGEN05", "lib", "metric_code", "default_context"]
