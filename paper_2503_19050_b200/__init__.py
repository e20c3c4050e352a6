"""paper_2503_19050_b200 -- B200-native (sm_100a) intra-stage tuning sweep of
Mist (arXiv 2503.19050) behind the C ABI declared in include/mist.h.

Importing the package does not touch the GPU.  ``mist`` loads libmist.so
(built in-tree by ``paper_2503_19050_b200.build``) and fails loudly when it
is missing; there is no CPU fallback.
"""
from . import mist  # noqa: F401
from .mist import (Context, MistError, Spec, mist_enumerate_space, mist_eval_stage_costs,  # noqa: F401
                   mist_eval_stage_costs_at, mist_nccl_unique_id, mist_pareto_frontier,
                   mist_sample_frontier)
