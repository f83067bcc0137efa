"""B200-native online hot path of arXiv 2504.16344 (block-Toeplitz F / F*
matvec, K^{-1} apply, posterior mean and QoI forecast).

The compute path is libltb.so (sm_100a CUDA kernels behind the C ABI in
include/ltb.h); this package is the host-side mirror of the reference's
``ltibayes`` C++ API.  See DESIGN.md.
"""
from ._lib import build, kernel_launches, last_error, load  # noqa: F401
from .matvec import (BlockSeries, BlockToeplitzKernel, CapacityError, ConfigError,  # noqa: F401
                     CudaError, IoError,
                     DimensionError, KernelTag, Layout, LayoutError, LtbError, MatvecPlan,
                     NumericalError, ObsSeries, QoISeries, ShardedMatvecPlan, SpaceTimeField, StateError,
                     algorithmic_bytes, dense_apply, reindex, reindex_device)
from .engine import InferenceEngine, MapResult, QoIPrediction, normal_quantile  # noqa: F401
from .artifacts import (Manifest, fnv1a64_file, infer_from_artifacts, read_manifest, read_series,  # noqa: F401
                        verify_manifest, write_dense, write_engine_artifacts, write_kernel, write_manifest,
                        write_series)
