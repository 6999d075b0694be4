"""B200-native (sm_100a) QUIK hybrid W4A4 / W8A8 linear layer.

Drop-in for the reference's C++ layer API (arXiv 2310.09259 reference,
proj/include/quik/runtime.hpp): the same functions over hand-written tcgen05/TMA
kernels behind the C ABI in include/quik_b200.h.
"""
from .quik import (  # noqa: F401
    ActQuantResult,
    BlockOp,
    Context,
    FormatError,
    NumericalError,
    load_layer,
    OutlierSet,
    PackedIntMatrix,
    PipelineVariant,
    QuantizedWeights,
    QuikGatedMLP,
    QuikLinear,
    QuikLinearLayer,
    StageTimes,
    compute_wreduced,
    dequantize_epilogue,
    dequantize_weights,
    forward_model,
    forward_model_trace,
    gated_mlp_ops,
    gptq_quantize_device,
    hessian_device,
    int_matmul,
    pack_values,
    quantize_activations,
    quantize_activations_fused,
    quik_matmul,
    row_bytes,
    rtn_quantize_weights,
    rtn_quantize_weights_device,
    split_activations,
    unpack_int4,
    unpack_values,
)
from ._lib import LIB_PATH, load as load_library  # noqa: F401

__version__ = "0.1.0"
