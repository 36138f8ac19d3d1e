"""B200-native KVLinC decode hot path (arXiv 2510.05373).

Drop-in replacement for the reference `quantkv` package's quantizer, cache
and attention API (names re-exported below, as in quantkv/__init__.py:4-19),
backed by hand-written sm_100a CUDA kernels in `libkvlinc.so` behind the C
ABI of `include/kvlinc.h`.  There is no CPU fallback: compute calls raise on
a host without a B200.

    import paper_2510_05373_b200 as quantkv     # instead of `import quantkv`

The batched serving path (B x Hkv caches, GQA decode, split-KV across GPUs)
is `paper_2510_05373_b200.batched` / `.distributed`.
"""
from .adapter import (CorrectionAdapter, correction_term, feature_map, phi_k, phi_q,  # noqa: F401
                      rng)
from .attention import (DecodePartial, OpCounter, attention_reference, attention_with_config,  # noqa: F401
                        corrected_attention_quadratic, corrected_attention_recurrent, decode_step_blocked,
                        quantize_roundtrip)
from .cache import (CacheFormatError, FootprintReport, KVCacheState, deserialize_cache,  # noqa: F401
                    memory_footprint, read_cache, serialize_cache, write_cache)
from .hadamard import HadamardMatrix, hadamard_matrix, rotate  # noqa: F401
from .linalg import matmul, softmax_rows  # noqa: F401
from .train import (AdamState, AdapterFormatError, TrainSettings, corrected_weights,  # noqa: F401
                    deserialize_adapter, loss_and_grads, read_adapter, serialize_adapter, train_adapter,
                    write_adapter)
from .quantize import (QuantConfig, QuantizedTensor, dequantize_group,  # noqa: F401
                       expected_quant_mse, pack_codes, quantize_group, quantize_tensor,
                       unpack_codes)

__version__ = "1.0.0"

__all__ = [
    "CorrectionAdapter", "correction_term", "feature_map", "phi_q", "phi_k", "rng",
    "DecodePartial", "decode_step_blocked", "quantize_roundtrip", "OpCounter", "attention_reference",
    "attention_with_config", "corrected_attention_quadratic", "corrected_attention_recurrent",
    "FootprintReport", "KVCacheState", "memory_footprint", "serialize_cache", "deserialize_cache",
    "read_cache", "write_cache", "CacheFormatError",
    "HadamardMatrix", "hadamard_matrix", "rotate", "matmul", "softmax_rows",
    "AdamState", "AdapterFormatError", "TrainSettings", "corrected_weights", "loss_and_grads", "train_adapter",
    "serialize_adapter", "deserialize_adapter", "read_adapter", "write_adapter",
    "QuantConfig", "QuantizedTensor", "dequantize_group", "expected_quant_mse", "pack_codes",
    "quantize_group", "quantize_tensor", "unpack_codes",
]
