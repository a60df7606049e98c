"""Exception types of the drop-in boundary.

Same names and base classes as the reference's ``admmprune.errors``
(/root/reference/pkg/src/admmprune/errors.py:4-13) so callers' ``except``
clauses keep working. The C ABI returns integer codes that map 1:1 onto these
(see include/hsx.h, ``HSX_E*``).
"""


class ShapeError(ValueError):
    """A tensor, mask, index set or layer table has a structurally invalid shape."""


class ProtocolError(RuntimeError):
    """A collective or cache was used inconsistently across ranks."""


class ConfigError(ValueError):
    """A configuration (penalties, topology, settings) is invalid."""


class CudaError(RuntimeError):
    """The CUDA runtime reported an error inside libhsx (code HSX_ECUDA)."""
