"""B200-native Torontonian engine (arxiv 2009.01177 hot path) behind the torfp API.

    import paper_2009_01177_b200 as torfp
    m = torfp.from_dense(O)                       # or load_matrix / generate_instance
    res = torfp.torontonian(m, precision="auto")  # GPU, DD/QD/fp64
"""
from .api import (device_count, det_i_minus_a, fold_partials, force_width, probability,
                  probability_reference, select_precision, torontonian, torontonian_batch,
                  torontonian_classes, torontonian_reference, torontonian_shard, torontonian_slice)
from .errors import (BreakdownError, DeviceError, InvalidArgument, ParseError, PrecisionError,
                     ResourceError, TorfpError)
from .matrix import (InputMatrix, check_symmetries, dequantize, extract_submatrix, from_dense,
                     load_matrix, quantize)
from .subsets import (binom, factorization_op_count, get_kth_mask, get_next_mask, partition,
                      prefix_classes, total_op_count)
from .workloads import generate_instance

__all__ = [
    "InputMatrix", "TorfpError", "InvalidArgument", "BreakdownError", "PrecisionError", "ParseError",
    "ResourceError", "DeviceError", "binom", "check_symmetries", "dequantize", "extract_submatrix",
    "factorization_op_count", "from_dense", "generate_instance", "get_kth_mask", "get_next_mask",
    "load_matrix", "partition", "prefix_classes", "probability", "probability_reference", "quantize",
    "select_precision", "force_width", "det_i_minus_a", "torontonian", "torontonian_reference",
    "torontonian_batch", "torontonian_slice", "torontonian_classes", "torontonian_shard", "fold_partials", "total_op_count",
    "device_count",
]

__version__ = "0.1.0"
