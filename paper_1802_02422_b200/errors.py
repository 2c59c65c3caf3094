"""Exception types of the reference (givf/errors.py:1-37) used by the path.

When the reference package is importable its classes are reused, so code
that catches `givf.errors.InvariantError` (or `StorageError`) keeps working
with this drop-in.
"""

try:  # pragma: no cover - depends on the caller's environment
    from givf.errors import (  # type: ignore
        BadMagicError,
        ChecksumError,
        GivfError,
        InvariantError,
        StorageError,
        VersionError,
    )
except Exception:  # noqa: BLE001

    class GivfError(Exception):
        pass

    class StorageError(GivfError):
        """Problem with a serialized index file."""

    class BadMagicError(StorageError):
        pass

    class VersionError(StorageError):
        pass

    class ChecksumError(StorageError):
        pass

    class InvariantError(GivfError):
        """An internal self-check failed; indicates a bug, not a usage error."""
