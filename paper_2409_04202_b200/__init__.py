"""B200-native GenModel/GenTree AllReduce (arXiv 2409.04202), C-ABI library + thin binding.

The compute path lives in `libgentree_ar.so` (include/gentree_ar.h): the planning core
(GenModel, GenTree Algorithms 1-2, fit) and the sm_100a executor kernels.  This package only
marshals arguments; importing it without the built library raises ImportError.
"""
from .api import (Comm, Executor, GmParams, Nvls, Plan, allreduce_exec, allreduce_exec_host, default_paths, dtype_code,  # noqa: F401
                  fill_synthetic, genmodel_closed_form, genmodel_fit, genmodel_fit_nvls, genmodel_fit_row, local_reduce, params,
                  rank_stride_bytes)
from ._lib import AR_BF16, AR_F32, ArError, ArInvalid, LIB_PATH  # noqa: F401
