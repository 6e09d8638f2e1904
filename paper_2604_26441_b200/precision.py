"""Per-level precision tags and BF16 rounding (reference: precision.py:1-48).

``round_bf16`` runs the round-to-nearest-even bit trick on the device
(``sg_vec_bf16``) for any array size; scalars are rounded the same way.
"""

from __future__ import annotations

import enum

import numpy as np

from . import _native

#: unit roundoff of BF16 (8-bit significand incl. the hidden bit)
EPS_BF16 = 2.0 ** -8


class PrecisionTag(enum.Enum):
    FP64 = "fp64"
    FP32 = "fp32"
    BF16EMU = "bf16"

    @property
    def working_dtype(self):
        """Smoother working dtype: float64 for FP64, float32 otherwise."""
        return np.float64 if self is PrecisionTag.FP64 else np.float32

    @property
    def code(self) -> int:
        return {"fp64": 0, "fp32": 1, "bf16": 2}[self.value]


def round_bf16(x):
    """Nearest BF16 value (ties to even) of the FP32 bit pattern; NaN kept.

    Float64 input is cast to float32 first.  Returns float32 (array input) or
    a Python float (scalar input), like the reference.
    """
    from . import _dev
    scalar = np.isscalar(x) or getattr(x, "ndim", 0) == 0
    t, host = _dev.as_device(np.reshape(np.asarray(x, dtype=np.float32), -1)
                             if not _dev.is_device_tensor(x) else x, np.float32)
    out = _dev.empty(t.numel(), np.float32)
    _native.call("sg_vec_bf16", t.numel(), _dev.ptr(t), _dev.ptr(out), _dev.stream())
    if scalar:
        return float(out.cpu().numpy()[0])
    res = _dev.back(out, host)
    if host:
        return res.reshape(np.shape(x))
    return res
