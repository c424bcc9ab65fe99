"""paper_2603_09632_b200 — B200-native X-GS hot path (VQ + voxel grid sampling).

A drop-in for the reference package ``semsplat``'s VQ and back-projection /
grid-sampling functions (same names and signatures), backed by hand-written
sm_100a CUDA kernels in ``_lib/libxgs.so`` (C ABI: include/xgs.h).
"""

from .core import CameraIntrinsics, CameraPose, Codebook, FeatureReservoir, GaussianField
from .errors import InvalidInputError, InvalidStateError, NativeError, SemsplatError
from .vq import (ReviveResult, VqAuditLog, VqBatchStats, VqConfig, WarmStartResult, accumulate, assign,
                 assign_batch, confidence_mask, confidence_scores, ema_step, online_step, revive_dead_codes,
                 seed_from_samples, squared_distances, warm_start)

__version__ = "0.1.0"
