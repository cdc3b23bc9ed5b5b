"""B200-native (sm_100a) TT-EmbeddingBag hot path of Rec-AD (arxiv 2507.14668).

Public surface:
    TTEmbeddingBag                 drop-in TT-compressed sum-pooled EmbeddingBag
    TtEngine                       one table's plan/forward/backward on the GPU
    geometry (TtShape, factorize_dims, ...), ops (reference operator API)
    build()                        compile libttb.so in-tree
"""
from .build import build  # noqa: F401
from .geometry import (TtShape, factorize_dims, init_random_cores, linear_index_to_tt_index,  # noqa: F401
                       param_stats, tt_index_to_linear)

__all__ = ["build", "TtShape", "factorize_dims", "init_random_cores", "linear_index_to_tt_index",
           "param_stats", "tt_index_to_linear", "TTEmbeddingBag", "TtEngine"]


def __getattr__(name):  # torch-dependent pieces load lazily
    if name == "TTEmbeddingBag":
        from .embedding_bag import TTEmbeddingBag
        return TTEmbeddingBag
    if name == "TtEngine":
        from .engine import TtEngine
        return TtEngine
    raise AttributeError(name)
