"""Exception classes of the engine.

Same names and meaning as the reference's hierarchy
(/root/reference/pkg/src/sentinel/errors.py:4-33) so ``except`` clauses written
against it keep working. ``raise_for_status`` turns a C-ABI status code
(include/sentinel_b200.h, ``snt_status``) into the matching class.
"""

from __future__ import annotations


class SentinelError(Exception):
    """Root of every error this package raises on purpose."""


class InvalidInput(SentinelError):
    """A precondition on an argument does not hold (empty model, zero blocks ...)."""


class InvalidState(SentinelError):
    """The object is not in a state the operation accepts (e.g. one digest left to reduce)."""


class ConfigError(SentinelError):
    """The hashing options contradict each other or are out of range."""


class FormatError(SentinelError):
    """A manifest, bundle or payload cannot be parsed."""


class ValidationError(SentinelError):
    """The data is well formed but semantically wrong (e.g. an undeclared source id)."""


class ResourceError(SentinelError):
    """A device, allocation or I/O resource is unavailable -- including a missing GPU or
    a missing native library: this engine has no CPU fallback."""


class KeyMaterialError(SentinelError):
    """Signing key material is absent, malformed or unusable."""


_STATUS_TO_EXC = {
    -1: InvalidInput,
    -2: InvalidState,
    -3: ConfigError,
    -4: ValidationError,
    -5: ResourceError,
}


def raise_for_status(status: int, what: str, detail: str = "") -> None:
    """Raise the exception class that corresponds to a negative ``snt_status``."""
    if status == 0:
        return
    exc = _STATUS_TO_EXC.get(status, SentinelError)
    msg = f"{what} failed (status {status})"
    if detail:
        msg += f": {detail}"
    raise exc(msg)
