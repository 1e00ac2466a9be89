"""B200-native Lightning Grasp forward pass (arXiv 2511.07418).

The hot path (contact-field build + query, contact search with the wrench
test, DLS-IK realisation + collision filter) runs as sm_100a kernels in
libgraspgen_b200.so behind the C-ABI in include/lg.h; this package is the
Python mirror of that boundary.  It holds no loader: hands, meshes, samples
and configs arrive as flat lg.h descriptors from the caller (the repository's
stand-in caller is the top-level `caller` package).
"""
from .api import (  # noqa: F401
    ContactFieldIndex, Context, CudaError, DevicePatches, RunResult, device_count,
    hand_patches_device, index_cache_key, lib, libm_eval, mix_seed, preprocess_object,
    query_domains_batch, run_batch, validate_batch, validation_issues,
)
from . import api  # noqa: F401
