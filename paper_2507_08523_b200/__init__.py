"""InferLog hot path on B200 (sm_100a): PAIR + prefix-cache-aware prefill.

The product is libinferlog_b200.so (include/il.h); this package is its thin binding.
Importing it does not load the library; Context / Pipeline do, and raise if it is missing.
"""
from ._lib import (IL_F_DEDUP, IL_F_EXCLUDE_SELF, IL_F_GUARD, IL_F_PAIR, IL_F_VERIFY, IL_SIM_COSINE, IL_SIM_JACCARD,
                   ILError, load)

__all__ = ["Config", "Context", "Pipeline", "ILError", "load", "IL_F_PAIR", "IL_F_GUARD",
           "IL_F_EXCLUDE_SELF", "IL_F_VERIFY", "IL_F_DEDUP", "IL_SIM_COSINE", "IL_SIM_JACCARD"]


def __getattr__(name):
    if name in ("Config", "Context"):
        from . import context
        return getattr(context, name)
    if name == "Pipeline":
        from .pipeline import Pipeline
        return Pipeline
    raise AttributeError(name)
