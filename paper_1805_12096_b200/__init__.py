"""B200-native batched greedy decoding of distilled Transformer / AAN students with
int8 tensor-core products (arXiv 1805.12096).  See DESIGN.md.

The compute path is libmnmt.so (sm_100a CUDA); this package is its binding plus the
multi-GPU driver (dist.py).  It never imports the CPU oracle.
"""
from .mnmt import (DEVICE_IO, DUMP_DEC_OUT, DUMP_ENC_OUT, DUMP_LAYERS, DUMP_OUT_CODES,  # noqa: F401
                   DUMP_SRC_KV, EXPORTS, LIB_PATH, MAX_SPAN, MnmtError, Model, batch_by_words,
                   lib)
