"""B200-native hot path of Photo-SLAM's photorealistic mapping (arXiv 2311.16728):
differentiable 3D Gaussian splatting render / loss / backward / pyramid / Adam as
hand-written sm_100a kernels behind the C ABI of include/gs.h (libgs.so)."""
from . import _lib  # noqa: F401
from .core import (Adam, AdamConfig, PhotometricLoss, Renderer, Workspace, gaussian_pyramid,  # noqa: F401
                   pack_params, param_rows, unpack)
from .mapping import MappingEngine, gp_level, reduce_gradients, shard_views  # noqa: F401
