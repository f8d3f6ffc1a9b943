"""Error types of the drop-in (reference: pkg/src/semcache/errors.py:6-23).

When the reference package `semcache` is importable, these classes
subclass its own, so callers that catch `semcache.errors.ValidationError`
(or `RetriableError`) keep working with the GPU path unchanged.
"""

from __future__ import annotations

try:  # pragma: no cover - depends on the caller's environment
    from semcache.errors import RetriableError as _RefRetriable
    from semcache.errors import SemcacheError as _RefBase
    from semcache.errors import ValidationError as _RefValidation
except Exception:  # noqa: BLE001
    _RefBase = Exception
    _RefValidation = None
    _RefRetriable = None


class SemcacheError(_RefBase):
    """Base class for errors raised by this package."""


if _RefValidation is not None:  # pragma: no cover
    class ValidationError(SemcacheError, _RefValidation):
        """Bad input: malformed value, dimension mismatch, unknown or duplicate id."""

    RetriableError = _RefRetriable
else:
    class ValidationError(SemcacheError):
        """Bad input: malformed value, dimension mismatch, unknown or duplicate id."""

    class RetriableError(SemcacheError):
        """Transient backend failure; the caller may retry."""
