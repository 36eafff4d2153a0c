"""Executor shim for the reference's dispatch argument.

The reference dispatches the spot body through
``parallel_for_blocks(executor, label, policy, body)`` on a thread pool
(/root/reference/pkg/src/xtrace/execution.py:66-125,207-224).  Here the
dispatch is one CUDA launch, so an executor only matters as the place where
callers read kernel timings (``kernel_timer``, execution.py:350-356).
``Executor.serial()`` / ``Executor.workers(n)`` are accepted so callers and
tests written against the reference run unchanged; every executor produces
the same bits because every pixel's accumulation is private and sequential.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Callable, NamedTuple

__all__ = ["Executor", "TimingRecord", "kernel_timer"]


class TimingRecord(NamedTuple):
    label: str
    ms: float


@dataclass
class Executor:
    kind: str = "serial"
    n: int = 1
    name: str = ""
    timing_log: list[TimingRecord] = field(default_factory=list)

    def __post_init__(self):
        if self.kind not in ("serial", "workers"):
            raise ValueError(f"unknown executor kind {self.kind!r}")
        if self.n < 1:
            raise ValueError("worker count must be >= 1")
        if self.kind == "serial":
            self.n = 1
        if not self.name:
            self.name = "serial" if self.kind == "serial" else f"workers{self.n}"

    @classmethod
    def serial(cls, name: str = "") -> "Executor":
        return cls("serial", 1, name)

    @classmethod
    def workers(cls, n: int | None = None, name: str = "") -> "Executor":
        return cls("workers", n or 1, name)

    @property
    def parallel(self) -> bool:
        return self.kind == "workers" and self.n > 1

    def close(self):
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def kernel_timer(executor: Executor, label: str, fn: Callable[[], object]):
    """Run fn, append (label, wall ms) to the executor's log, return fn's result."""
    t0 = time.perf_counter()
    try:
        return fn()
    finally:
        executor.timing_log.append(TimingRecord(label, (time.perf_counter() - t0) * 1e3))
