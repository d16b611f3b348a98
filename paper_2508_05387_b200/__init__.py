"""paper_2508_05387_b200 -- B200-native learner hot path of Echo (arXiv 2508.05387).

The product is libecho.so (CUDA for sm_100a, C ABI in include/echo.h).  This package holds its sources
(csrc/), the in-tree build (_build.py), the ctypes binding (abi.py, same names as the C ABI), the
per-rank step driver (step.py) and the data-parallel plumbing (parallel.py).
"""
from . import abi  # noqa: F401  (raises ImportError when libecho.so is missing: no fallback path)
from .abi import (EchoError, echo_abi_version, echo_group_advantage, echo_loss_stats,  # noqa: F401
                  echo_loss_stats_workspace_bytes, echo_pack_batch, echo_policy_loss_fwd_bwd, echo_status_string)
