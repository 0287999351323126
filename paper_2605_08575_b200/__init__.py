"""B200-native activation-sparse MoE FFN layer (drop-in for the `sparsekit` layer API).

The package is a thin host-side mirror of the reference interface over
``lib/libsparsekit_b200.so`` (hand-written sm_100a CUDA behind the C ABI declared in
``include/sparsekit_b200.h``).  Importing it loads the library; a missing build is an error.
"""
from . import _lib

_lib.load()  # fail loudly when the CUDA library has not been built

from .layer import *  # noqa: E402,F401,F403
from .layer import (MoEConfig, MoELayerWeights, SparsityLevel, forward_dense,  # noqa: E402,F401
                    forward_masked_dense, forward_sparse, forward_topk_sparse)
