"""B200-native Lightning Grasp forward pass (arXiv 2511.07418).

The hot path (contact-field build + query, contact search with the wrench
test, DLS-IK realisation + collision filter) runs as sm_100a kernels in
libgraspgen_b200.so behind the C-ABI in include/lg.h; this package is the
Python mirror of the reference's C++ API over that boundary.
"""
from .api import (  # noqa: F401
    ContactFieldIndex, Context, CudaError, HandModel, Mesh, Patches, RunResult,
    default_config, device_count, hand_patches, hand_patches_device, index_cache_key, lib, load_hand, load_mesh,
    mix_seed, parse_config, prepare_inputs, preprocess_object, query_domains_batch, run_batch,
    sample_surface, validate_batch, validation_issues, write_dataset, write_profile,
)
