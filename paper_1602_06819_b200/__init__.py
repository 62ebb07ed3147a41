"""B200-native online approximate k-nn graph (arXiv 1602.06819): iGNNS search + depth-bounded
reverse update in batches, behind the C ABI of include/knng.h (libknng.so, sm_100a)."""
from .knng import (KnngGraph, KnngError, TokenSets, load_library, nccl_unique_id, EXPORTS, KNNG_L2SQ_U8, KNNG_L2SQ_F32,
                   KNNG_JACCARD_U32SET, KNNG_JARO_WINKLER, KNNG_COSINE_2GRAM, Strings, LIB_PATH)

__all__ = ["KnngGraph", "KnngError", "TokenSets", "load_library", "nccl_unique_id", "EXPORTS", "KNNG_L2SQ_U8", "KNNG_L2SQ_F32",
           "KNNG_JACCARD_U32SET", "KNNG_JARO_WINKLER", "KNNG_COSINE_2GRAM", "Strings", "LIB_PATH"]
