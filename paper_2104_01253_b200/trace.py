"""Lightweight launch tracing (SURVEY.md §5 "Tracing / profiling").

When a Recorder is active, the engine and the operators report every kernel
launch with its algorithmic HBM bytes, and (optionally) bracket the hot
kernels and the cross-rank allreduce with CUDA events on the launching
stream.  With no recorder active the hooks cost one attribute check.
"""

import contextlib
from collections import defaultdict

import torch

_active = None


class Recorder:
    def __init__(self, events=False):
        self.events = events
        self.calls = defaultdict(int)
        self.bytes = defaultdict(int)
        self._spans = defaultdict(list)

    def note(self, name, nbytes):
        self.calls[name] += 1
        self.bytes[name] += int(nbytes)

    @contextlib.contextmanager
    def span(self, name):
        if not self.events:
            yield
            return
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        try:
            yield
        finally:
            e.record()
            self._spans[name].append((s, e))

    def seconds(self, name):
        """Summed device time of a span kind (synchronizes)."""
        torch.cuda.synchronize()
        return sum(s.elapsed_time(e) for s, e in self._spans[name]) * 1e-3

    def span_count(self, name):
        return len(self._spans[name])

    def total_bytes(self):
        return sum(self.bytes.values())

    def total_calls(self):
        return sum(self.calls.values())


def start(events=False):
    global _active
    _active = Recorder(events)
    return _active


def stop():
    global _active
    rec, _active = _active, None
    return rec


def note(name, nbytes):
    if _active is not None:
        _active.note(name, nbytes)


@contextlib.contextmanager
def span(name):
    if _active is None or not _active.events:
        yield
    else:
        with _active.span(name):
            yield
