"""Exception types of the reference (givf/errors.py:1-37) used by the path.

When the reference package is importable its classes are reused, so code
that catches `givf.errors.InvariantError` keeps working with this drop-in.
"""

try:  # pragma: no cover - depends on the caller's environment
    from givf.errors import GivfError, InvariantError  # type: ignore
except Exception:  # noqa: BLE001

    class GivfError(Exception):
        pass

    class InvariantError(GivfError):
        """An internal self-check failed; indicates a bug, not a usage error."""
