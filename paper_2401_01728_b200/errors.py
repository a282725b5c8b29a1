"""Exception classes of the averaging path.

Names and meanings follow the reference hierarchy
(/root/reference/pkg/src/ravnest/errors.py:4-65) so callers that catch the
reference's exceptions keep working: C-ABI status codes map onto these in
``_native.check``.  When the reference package is importable, ``plugin.install``
aliases these names to the reference's own classes.
"""


class RavnestError(Exception):
    """Root of every error raised on the averaging path."""


class ConfigError(RavnestError):
    """Unusable configuration, e.g. fewer than two clusters (multiring.py:268-269)."""


class LayoutError(RavnestError):
    """Cluster layouts or vectors disagree about the parameter space
    (multiring.py:64-131, 270-275)."""


class ProtocolError(RavnestError):
    """A message or state transition the ring protocol forbids (multiring.py:207-211)."""


class StallError(RavnestError):
    """A cycle could not complete: a peer never reached a barrier
    (multiring.py:296-298; here a device-side flag timeout)."""


class SchemaError(RavnestError):
    """A file whose schema tag or layout the reader does not accept
    (configio.py:195-198, 505-510)."""
