"""B200-native HiNM (arXiv 2407.20496) hot path behind the reference ``hinm`` API.

Drop-in names (same meaning, arguments and exceptions as the reference package):
HiNMConfig, validate_config, GyroPermutation, MaskPair, magnitude_saliency, vector_prune,
nm_prune, encode, decode, restore_row_order, hinm_spmm, HiNMEncoding, TileEncoding, errors.
Device-level API: ``compress`` (fused GPU compressor -> DevicePack) and ``spmm`` (tcgen05).
"""

from .errors import (BudgetError, CapacityError, CountError, DeviceError, DimensionError,
                     FormatError, GroupingError, HiNMError, InvariantViolation, NegativeScore,
                     ShapeMismatch, SizeGuard, exit_code_for)
from .model import (DenseMatrix, GyroPermutation, HiNMConfig, MaskPair, SaliencyMatrix,
                    ValidatedConfig, composed_sparsity, count_permutation_space,
                    default_sample_schedule, identity_permutation, validate_config)
from .pruning import (HiNMEncoding, TileEncoding, apply_masks, decode, encode, encoding_from_pack,
                      load_saliency, magnitude_saliency, masked_dense_from_encoding, nm_prune,
                      restore_row_order, survivors_per_tile, validate_masks, vector_prune)
from .spmm import (LayerChain, TileBuffer, build_layer_chain, compose_layers, dense_matmul,
                   gather_tile_buffer, hinm_spmm, hinm_spmm_original_order, kept_triples,
                   relative_error, shuffle_encoding, tile_shuffle_check)
from .permutation import (Partition, PruneReport, ScheduleState, ablation_mode, assignment_cost,
                          balanced_kmeans, gyro_permute, hungarian, icp_tile, no_perm_prune,
                          ocp_iterate, retained_saliency, sample_channels)
from . import io
from .device import (DevicePack, HostChain, build_group_image, build_operand_image, compress,
                     compress_layers, spmm, spmm_simt)

__version__ = "0.1.0"

__all__ = [
    "BudgetError", "CapacityError", "CountError", "DeviceError", "DimensionError", "FormatError",
    "GroupingError", "HiNMError", "InvariantViolation", "NegativeScore", "ShapeMismatch",
    "SizeGuard", "exit_code_for", "DenseMatrix", "GyroPermutation", "HiNMConfig", "MaskPair",
    "SaliencyMatrix", "ValidatedConfig", "composed_sparsity", "count_permutation_space",
    "default_sample_schedule",
    "identity_permutation", "validate_config", "HiNMEncoding", "TileEncoding", "apply_masks",
    "decode", "encode", "encoding_from_pack", "load_saliency", "magnitude_saliency",
    "masked_dense_from_encoding", "nm_prune", "restore_row_order", "survivors_per_tile",
    "validate_masks", "vector_prune", "TileBuffer", "dense_matmul", "gather_tile_buffer",
    "hinm_spmm", "hinm_spmm_original_order", "relative_error", "DevicePack",
    "build_operand_image", "build_group_image", "compress", "compress_layers", "spmm",
    "spmm_simt", "HostChain", "LayerChain",
    "build_layer_chain", "compose_layers", "kept_triples", "shuffle_encoding",
    "tile_shuffle_check", "no_perm_prune", "io", "PruneReport", "ablation_mode",
    "balanced_kmeans", "gyro_permute", "hungarian", "icp_tile", "ocp_iterate",
    "retained_saliency", "sample_channels", "Partition", "ScheduleState", "assignment_cost",
]
