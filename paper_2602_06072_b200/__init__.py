"""B200-native PackInfer hot path (arXiv 2602.06072): C ABI library + thin Python binding.

The product path is libpackinfer.so (include/packinfer.h); this package only marshals arguments.
It never imports the test oracle and has no CPU fallback.
"""

from .packinfer import (  # noqa: F401
    PackInferError, PackedBatch, default_config, lib, packinfer_attention_decode,
    packinfer_attention_prefill, packinfer_merge, packinfer_plan, packinfer_plan_upload,
    packinfer_relayout_kv, version,
)
