"""paper_2204_05496_b200 — B200-native (sm_100a) encrypted logistic-regression
matmul hot path of arXiv 2204.05496 (fast slot-packed algorithm + standard
sample-batched comparator), behind the reference's hei::matmul interface.

The compute path is libheinfer_b200.so (hand-written CUDA, C ABI in
include/heinfer_b200.h); this package is the Python host mirror.
"""
from .native import (  # noqa: F401
    CodecError,
    CudaError,
    FORM_COEFF,
    FORM_EVAL,
    KeyError_,
    NativeLibraryError,
    NoiseError,
    OpCounters,
    ParamError,
    RangeError,
)
from .matmul import (  # noqa: F401
    EncodedWeights,
    GpuTwinServer,
    MatmulStream,
    Prng,
    baseline_matmul,
    ScalingConfig,
    baseline_counts,
    encode_bias,
    encode_inputs,
    encode_inputs_device,
    encode_weights,
    matmul,
    matmul_device,
    matmul_wire,
    save_ciphertexts,
    default_q_primes,
    proposed_counts,
    scale_value,
)
