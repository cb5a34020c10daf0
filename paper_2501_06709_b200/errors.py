"""Exception hierarchy of the drop-in API.

Same class names and base-class relations as the reference's
(/root/reference/pkg/src/kvpack/errors.py:4-32) so `except ConfigError`
etc. keep working for callers that switch packages, plus two data-plane
errors for failures the reference cannot have (it moves no bytes).
"""
from __future__ import annotations


class KvPackError(Exception):
    """Root of every error this package raises on purpose."""


class RequestTooLarge(KvPackError):
    """A request's KV footprint does not fit one GPU (errors.py:8-9)."""


class NotPlaced(KvPackError):
    """Unknown request / item / pool (errors.py:12-13)."""


class NoCategory(KvPackError):
    """An empty GPU has no size category (errors.py:16-17)."""


class ConfigError(KvPackError):
    """Invalid topology, budget or pool geometry (errors.py:20-21)."""


class ParseError(KvPackError):
    """Malformed trace row; keeps the 1-based line number (errors.py:24-32)."""

    def __init__(self, message, line=None):
        text = message if line is None else f"line {line}: {message}"
        super().__init__(text)
        self.line = line


class KvmCudaError(KvPackError):
    """A CUDA runtime call inside libkvmig failed (KVM_ERR_CUDA)."""


class KvmUnsupported(KvPackError):
    """The native library lacks a feature or the device is not sm_100."""


class NativeLibraryMissing(KvPackError, ImportError):
    """libkvmig.so is not built.  There is deliberately no CPU fallback."""
