"""B200-native patch featurization + threshold similarity join.

A drop-in for the data-parallel hot path of the reference ``patchdb``
engine (DeepLens, arXiv 1812.07607): colour-histogram featurization of
uint8 frame tiles and the threshold similarity join over the features.
The compute runs in hand-written sm_100a kernels behind the C-ABI of
include/pdb_cuda.h (libpdb_cuda.so); this package is the host-side mirror
of the reference operator interface (see patchdb.py).
"""

from . import _capi, patchdb, workloads  # noqa: F401
from .patchdb import (  # noqa: F401
    BuildSide, ConfigError, DeviceError, DimensionMismatchError, DuplicatePatchIdError, Error,
    Frame, GeneratorSpec, MixedDimensionError, Patch, ShapeError, TransformerSpec,
    apply_transformer, color_histogram, featurize_join, featurize_tiles, generate, sim_join,
    sim_join_device, sim_join_pairs, transform,
)

__version__ = "0.1.0"
