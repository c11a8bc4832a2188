"""paper_2507_03836_b200 -- B200-native (sm_100a) hot path of F-Hash
(arXiv 2507.03836): multi-resolution Tesseract encode through the paper's
MPHF, forward/backward, behind the C ABI in include/fhash.h.

The CUDA library is required: importing the binding does not fall back to
any CPU implementation.
"""
from .fhash import (Encoder, FHashError, fold_schedule, lib, FH_OK, FH_E_ARG, FH_E_RANGE, FH_E_DOMAIN,
                    FH_E_CUDA, FH_E_DIVERGED, FH_E_STATE, EXPORTS, LIB_PATH)

__all__ = ["Encoder", "FHashError", "fold_schedule", "lib", "EXPORTS", "LIB_PATH"]
