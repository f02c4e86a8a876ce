"""Engine error types of the drop-in boundary.

The C-ABI returns the status codes of include/forkattn.h; they surface here
as the reference's own exception classes (semflow/errors.py:71-84) whenever
the reference runtime is importable, so `except OutOfMemory` in the
reference manager (manager.py:488) catches errors raised by the GPU engine.
Without the reference package the classes below carry the same names and the
same stable `.code` strings (errors.py:10-18), which the HTTP layer maps to
status codes (api.py:37-56).
"""

from __future__ import annotations

try:  # the reference runtime is the caller; share its exception identity
    from semflow.errors import (  # type: ignore
        ContextBusy,
        OutOfMemory,
        SemflowError,
        UnknownContext,
        UnknownParentContext,
    )

    REFERENCE_ERRORS = True
except Exception:  # standalone (e.g. the GPU box, where semflow is absent)
    REFERENCE_ERRORS = False

    class SemflowError(Exception):  # type: ignore[no-redef]
        """Base class; `code` is the stable machine-readable name."""

        code = "internal"

        def __init__(self, message: str = "", **details):
            super().__init__(message or self.__class__.__name__)
            self.message = message or self.__class__.__name__
            self.details = details

    class OutOfMemory(SemflowError):  # type: ignore[no-redef]
        code = "out_of_memory"

    class UnknownContext(SemflowError):  # type: ignore[no-redef]
        code = "unknown_context"

    class UnknownParentContext(SemflowError):  # type: ignore[no-redef]
        code = "unknown_parent_context"

    class ContextBusy(SemflowError):  # type: ignore[no-redef]
        code = "context_busy"


class KernelError(SemflowError):
    """A CUDA failure or misuse of the device path (C-ABI codes 5-7)."""

    code = "internal"


__all__ = [
    "SemflowError",
    "OutOfMemory",
    "UnknownContext",
    "UnknownParentContext",
    "ContextBusy",
    "KernelError",
    "REFERENCE_ERRORS",
]
