"""LosslessPredictor codec (proj/src/codec_kernels.hpp:165-239) on the GPU.

SURVEY.md §8(f) row 1 ("next"): not built yet.  Collectives routed through a
lossless CodecSpec still run (the codec is value-transparent, so the ring
moves raw fp32 through the identity kernels); standalone compress/decompress
of the predictor format raise UnsupportedError until the device codec lands.
"""
from __future__ import annotations

from .errors import UnsupportedError


def compress(buf):
    raise UnsupportedError("lossless predictor codec has no device implementation yet")


def decompress(cbuf):
    raise UnsupportedError("lossless predictor codec has no device implementation yet")
