"""volkrig-b200: B200-native kriging interpolation path of arXiv 2303.09523.

Drop-in for the reference's ``volkrig.kriging`` entry points, backed by
hand-written sm_100a CUDA kernels behind a C ABI (``include/volkrig_b200.h``).
"""

from .errors import (DegenerateLags, DeviceError, DeviceUnsupported,
                     InsufficientSamples, NoKnownNeighbors, SingularSystem,
                     TooFewSlices, VolkrigError)
from .model import SliceStack, VolumeGrid, missing_planes_per_gap
from .kriging import (KrigingPlan, VariogramModel, fill_missing, fit_variogram,
                      interpolate_voxel, solve_systems)
from .block_pipeline import ZPartKriging, reconstruct_zparts, subpart_ranges
from .blocks import BlockDescriptor, BlockKriging, partition, reconstruct_blocks
from .volume_io import load_volume, save_volume
from .stack_io import StackManifest, load_stack, normalize_stack, parse_manifest, write_manifest

__all__ = [
    "DegenerateLags", "DeviceError", "DeviceUnsupported", "InsufficientSamples",
    "NoKnownNeighbors", "SingularSystem", "TooFewSlices", "VolkrigError",
    "SliceStack", "VolumeGrid", "missing_planes_per_gap", "KrigingPlan",
    "VariogramModel", "fill_missing", "fit_variogram", "interpolate_voxel", "solve_systems",
    "ZPartKriging",
    "reconstruct_zparts", "subpart_ranges", "BlockDescriptor", "BlockKriging", "partition",
    "reconstruct_blocks", "load_volume", "save_volume", "StackManifest", "load_stack",
    "normalize_stack", "parse_manifest", "write_manifest",
]
