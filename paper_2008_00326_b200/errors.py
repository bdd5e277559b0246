"""Exception hierarchy of the drop-in boundary.

Mirrors the names raised by the reference on this path
(reference: pkg/src/rvpose/errors.py:4-61) so callers can keep their
``except`` clauses; `DeviceError` is new and covers CUDA / C-ABI failures.
"""


class RvposeError(Exception):
    pass


def _mk(name, doc):
    return type(name, (RvposeError,), {"__doc__": doc})


NonPositiveDepth = _mk("NonPositiveDepth", "camera-frame point with z <= 0")
InvalidDepth = _mk("InvalidDepth", "depth is non-positive, non-finite or invalid")
EmptyMesh = _mk("EmptyMesh", "mesh without triangles")
DimensionMismatch = _mk("DimensionMismatch", "image/array sizes disagree")
UnknownObjectId = _mk("UnknownObjectId", "object id has no registered model")
OutOfGamutInput = _mk("OutOfGamutInput", "sRGB component outside [0, 1]")
TooFewPoints = _mk("TooFewPoints", "cloud smaller than the neighbourhood size")
InvalidSpec = _mk("InvalidSpec", "malformed primitive or scene specification")
NoValidDepth = _mk("NoValidDepth", "detection mask without a valid-depth pixel")
EmptyBatch = _mk("EmptyBatch", "batch reduction over an empty collection")
EmptyModel = _mk("EmptyModel", "model point set is empty")
EmptyInput = _mk("EmptyInput", "metric over an empty error list")
ConfigError = _mk("ConfigError", "invalid search configuration")
DatasetError = _mk("DatasetError", "scene or model files missing or malformed")
DeviceError = _mk("DeviceError", "CUDA / libpx failure (no CPU fallback exists)")
