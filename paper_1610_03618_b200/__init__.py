"""B200-native (sm_100a) memory-bound CNN layer path of arXiv 1610.03618.

Layout transforms (NCHW<->CHWN), max/avg pooling in both layouts with
register coarsening, the fused softmax classifier and the paper's per-layer
layout selector, behind the reference's lcnn operator API.  The compute path
is hand-written CUDA in ``csrc/`` exposed through the C ABI of
``include/lcnn_cuda.h`` (``lib/liblcnn_cuda.so``); ``capi`` binds it and
``lcnn`` mirrors the reference operator API on device tensors.  The layout
selector and the network runtime are C++ (``host/``: the reference's
``lcnn::`` headers over the C ABI, ``lib/liblcnn.so``, C ABI in
``include/lcnn_net.h``); ``netapi`` binds that, ``shard`` holds the N-sharding
helpers of the multi-GPU runs.
"""
from . import errors  # noqa: F401
from .capi import CHWN, HWCN, NCHW, NHWC  # noqa: F401

__version__ = "0.1.0"
