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

    @classmethod
    def from_tally(cls, tally, pixels: int) -> "OpCounters":
        """Build from a flat tally array in the reference's slot order
        (col_add, col_cmp, win_add, win_cmp, ext_add, ext_cmp, elementary,
        replay, rebuild; counters.py:18-27)."""
        names = [f.name for f in fields(cls)][:9]
        return cls(**{k: int(tally[i]) for i, k in enumerate(names)}, pixels=int(pixels))

    def csv_row(self, label: str) -> str:
        """One row in the CSV_HEADER schema (counters.py:105-118)."""
        return ",".join([label] + [str(v) for v in (
            self.col_add, self.col_cmp, self.win_add, self.win_cmp, self.ext_add, self.ext_cmp,
            self.total_add, self.total_cmp)] + [f"{self.elementary_fraction:.6f}", str(self.pixels)])


CSV_HEADER = ("label,col_add,col_cmp,win_add,win_cmp,ext_add,ext_cmp,"
              "total_add,total_cmp,elementary_fraction,pixels")


def counters_report(rows, fmt: str = "human") -> str:
    """Render ``(label, OpCounters)`` rows as the reference's aligned
    per-pixel table (``"human"``) or CSV (counters.py:121-155)."""
    rows = list(rows)
    if fmt == "csv":
        return "\n".join([CSV_HEADER] + [c.csv_row(label) for label, c in rows])
    if fmt != "human":
        raise ValueError(f"unknown report format: {fmt!r}")
    lw = max([len(label) for label, _ in rows] + [9])
    out = [
        f"{'':{lw}}  {'columns':>15}  {'window':>15}  {'extraction':>15}  {'overall':>15}  {'elem%':>6}",
        f"{'per pixel':{lw}}  " + "  ".join(f"{'add':>7} {'cmp':>7}" for _ in range(4)) + f"  {'':>6}",
    ]
    for label, c in rows:
        p = c.pixels or 1
        pairs = ((c.col_add, c.col_cmp), (c.win_add, c.win_cmp), (c.ext_add, c.ext_cmp),
                 (c.total_add, c.total_cmp))
        out.append(f"{label:{lw}}  " + "  ".join(f"{a / p:7.2f} {b / p:7.2f}" for a, b in pairs)
                   + f"  {100.0 * c.elementary_fraction:5.1f}%")
    return "\n".join(out)
