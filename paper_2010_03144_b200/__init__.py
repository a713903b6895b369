"""paper_2010_03144_b200 -- B200-native SDC-resilient error-bounded lossy compressor.

Drop-in for the reference `ftlz` compress -> serialize / parse -> decompress path
(reference __init__.py:6-81): same names, argument meanings and exceptions, with every
stage running as hand-written sm_100a CUDA kernels behind the C ABI in include/ftlz_b200.h.
"""

from .core import (
    EB_ABSOLUTE,
    EB_RELATIVE,
    BlockGrid,
    BlockSpec,
    ErrorBound,
    Field,
    partition,
    resolve_error_bound,
)
from .container import BlockRecord, CompressedStream, parse, serialize
from .errors import (
    BackendUnavailable,
    BlockTooLarge,
    CorruptStream,
    DegenerateBound,
    DeviceError,
    FtlzError,
    InternalInvariantViolation,
    InvalidArgument,
    InvalidGeometry,
    InvalidInjection,
    InvalidRegion,
    IoError,
    ShapeMismatch,
    UncorrectableCorruption,
    UnsupportedCodec,
)
from .pipeline import (
    FtConfig,
    FtReport,
    compress,
    compress_bytes,
    cr_decrease_bound,
    decompress,
    decompress_bytes,
    decompress_region,
    intersecting_block_count,
)
from .predict import PredictorKind, RegressionCoeffs
from .quantize import QuantConfig
from .faults import CampaignReport, InjectionPlan, inject_bitflip, run_campaign, run_trial

__version__ = "0.1.0"

__all__ = [
    "BackendUnavailable", "BlockGrid", "CampaignReport", "InjectionPlan", "inject_bitflip",
    "run_campaign", "run_trial", "BlockRecord", "BlockSpec", "BlockTooLarge",
    "CompressedStream", "CorruptStream", "DegenerateBound", "DeviceError", "EB_ABSOLUTE",
    "EB_RELATIVE", "ErrorBound", "Field", "FtConfig", "FtReport", "FtlzError",
    "InternalInvariantViolation", "InvalidArgument", "InvalidGeometry", "InvalidInjection",
    "InvalidRegion", "IoError", "PredictorKind", "QuantConfig", "RegressionCoeffs",
    "ShapeMismatch", "UncorrectableCorruption", "UnsupportedCodec", "compress",
    "compress_bytes", "cr_decrease_bound", "decompress", "decompress_bytes", "decompress_region",
    "intersecting_block_count", "parse",
    "partition", "resolve_error_bound", "serialize",
]
