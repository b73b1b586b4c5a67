"""Exception taxonomy — the same names and bases as the reference
(errors.py:4-53), so `except mpc3.RangeError` code ports unchanged.  The C ABI
returns integer statuses that map 1:1 onto these (include/mpc3_b200.h)."""


class Mpc3Error(Exception):
    """Root of every engine error."""


def _kind(name: str, base: type, doc: str) -> type:
    return type(name, (Mpc3Error, base), {"__doc__": doc, "__module__": __name__})


RangeError = _kind("RangeError", ValueError, "Value outside the encodable / supported range (status 1).")
ShapeError = _kind("ShapeError", ValueError, "Incompatible tensor geometry (status 2).")
ExactnessError = _kind("ExactnessError", ValueError, "Accumulation beyond the exactness budget (status 3).")
ThresholdError = _kind("ThresholdError", ValueError, "Too few shares to reconstruct.")
IntegrityError = _kind("IntegrityError", ValueError, "Replicated components disagree (status 7).")
FreshnessError = _kind("FreshnessError", ValueError, "PRF (key, purpose, counter) reuse (status 5).")
TopologyError = _kind("TopologyError", ValueError, "Invalid party / peer (status 6).")
TransportError = _kind("TransportError", IOError, "Channel failure.")
FrameError = _kind("FrameError", ValueError, "Malformed wire frame.")
FormatError = _kind("FormatError", ValueError, "Malformed model / weight file.")
ConfigError = _kind("ConfigError", ValueError, "Invalid protocol or run configuration (status 4).")
ProtocolError = _kind("ProtocolError", RuntimeError, "Protocol-level failure during a run.")

__all__ = [
    "Mpc3Error", "RangeError", "ShapeError", "ExactnessError", "ThresholdError", "IntegrityError",
    "FreshnessError", "TopologyError", "TransportError", "FrameError", "FormatError", "ConfigError",
    "ProtocolError",
]
