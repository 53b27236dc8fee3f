"""paper_1910_06591_b200 — SEED (arXiv 1910.06591) learner / inference hot path on B200.

Thin Python binding over libseed.so (include/seed.h): argument marshalling
only — every step of the path runs in the library's sm_100a kernels.  Torch is
used for device memory, streams and process groups.
"""
from ._lib import SeedError, load  # noqa: F401
from .api import (  # noqa: F401
    HParams, Learner, InferenceServer, NetSpec, ParamSnapshot, PrioritizedReplay, r2d2_targets,
    R2d2HParams, R2d2Learner, debug_gemm, net_param_count, net_param_layout,
    spec_for_config, vtrace, Comm,
)
