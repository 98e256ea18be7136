"""OpCounters: the reference's reporting struct (pkg/src/medtree/counters.py:40-118).

The tallies count operations of the CPU tree algorithm (column/window/
extraction additions and comparisons); the GPU kernels run a different
algorithm, so the drop-in reports the reference's ``counting=False`` view:
all tallies zero and ``pixels`` = output pixels (SURVEY.md section 2 row 6,
reference tests/test_engine.py:226-240).
"""

from __future__ import annotations

from dataclasses import dataclass, fields


@dataclass
class OpCounters:
    col_add: int = 0
    col_cmp: int = 0
    win_add: int = 0
    win_cmp: int = 0
    ext_add: int = 0
    ext_cmp: int = 0
    elementary: int = 0
    replay: int = 0
    rebuild: int = 0
    pixels: int = 0

    def __add__(self, other: "OpCounters") -> "OpCounters":
        if not isinstance(other, OpCounters):
            return NotImplemented
        return OpCounters(**{f.name: getattr(self, f.name) + getattr(other, f.name)
                             for f in fields(self)})

    @property
    def total_add(self) -> int:
        return self.col_add + self.win_add + self.ext_add

    @property
    def total_cmp(self) -> int:
        return self.col_cmp + self.win_cmp + self.ext_cmp

    @property
    def sync_events(self) -> int:
        return self.elementary + self.replay + self.rebuild

    @property
    def elementary_fraction(self) -> float:
        events = self.sync_events
        return self.elementary / events if events else 0.0

    def per_pixel(self, field: str) -> float:
        value = getattr(self, field)
        return value / self.pixels if self.pixels else 0.0
