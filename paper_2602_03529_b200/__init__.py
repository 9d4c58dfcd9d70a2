"""B200-native (sm_100a) implementation of the semstream / Morphe codec hot
path: encoder -> 8-bit token quantisation -> priority packetisation with
intelligent dropping -> mask-aware decoder -> upscale + boundary blend.

The public names mirror the reference package's hot-path API
(/root/reference/pkg/src/semstream/__init__.py:6-24 and the codec / selection
/ transport modules) so this package is a drop-in for that path.  Every
numeric result comes from the CUDA kernels behind the C ABI in
include/semstream_b200.h; there is no CPU fallback.
"""

__version__ = "0.1.0"

from .codec import (BLOCK, COEFF_POSITIONS, CodecConfig, TokenMatrix, apply_token_mask,
                    bilinear_upscale, blend_boundary, decode_gop, downscale_frame, encode_gop,
                    scale_gop, token_grid_shape, upscale_frame)
from .selection import (DROP_RATE_CAP, LOSS_TOLERANCE, SimilarityMap, build_drop_mask,
                        drop_rate_for_bandwidth, token_similarity, top_k_drop_mask)
from .transport import (PacketFormatError, TokenPacket, packetize_tokens, parse_packet,
                        parse_packets, reassemble, token_packet_wire_size)
from .video import (GOP_SIZE, Frame, GoP, QualityReport, boundary_flicker, gop_psnr, mse, psnr,
                    segment_gops)
from .plugin import tokenizer_decode, tokenizer_encode
from .residual import (SparseResidual, aggregate_residual, apply_residual, compute_residual,
                       fit_to_budget, raw_residual_rate, sparsify_quantize)

__all__ = [
    "__version__",
    "BLOCK", "COEFF_POSITIONS", "CodecConfig", "DROP_RATE_CAP", "Frame", "GOP_SIZE", "GoP",
    "LOSS_TOLERANCE", "PacketFormatError", "QualityReport", "SimilarityMap", "TokenMatrix",
    "TokenPacket", "apply_token_mask", "bilinear_upscale", "blend_boundary", "boundary_flicker",
    "build_drop_mask", "decode_gop", "downscale_frame", "drop_rate_for_bandwidth", "encode_gop",
    "gop_psnr", "mse", "packetize_tokens", "parse_packet", "parse_packets", "psnr",
    "reassemble", "scale_gop", "segment_gops", "token_grid_shape", "token_packet_wire_size",
    "token_similarity", "tokenizer_decode", "tokenizer_encode", "top_k_drop_mask",
    "upscale_frame", "SparseResidual", "aggregate_residual", "apply_residual",
    "compute_residual", "fit_to_budget", "raw_residual_rate", "sparsify_quantize",
]
