"""Device event trace of the fused kernels (SURVEY §5 tracing; SPEC S:418-447 TraceEvent /
analyze_trace): read the records the kernels append when the "trace_events" option is set, convert
them to SPEC-format JSON Lines events, and summarise them (per rank and unit busy / wait time,
pairing diagnostics, and the communication time that overlaps computation).  Host-side plumbing:
no arithmetic of the method."""
from __future__ import annotations

import ctypes as C
import json

import numpy as np

from ._lib import check, lib

UNITS = ("compute", "copy")
KINDS = ("tile_start", "tile_end", "wait_start", "wait_end", "notify", "copy_start", "copy_end", "sm_clock")
_REC = np.dtype([("t_ns", "<u8"), ("tile", "<u4"), ("rank", "<u2"), ("unit", "u1"), ("kind", "u1")])


def read_events(comm, cap: int | None = None, clocks: bool = False):
    """Drain the comm's device trace into a list of SPEC TraceEvent dicts
    {"rank", "unit", "kind", "tile", "channel", "t_ns"} (+ "peer" for copy / notify events),
    sorted by time.  `channel` is left None: it follows from the tile through the static mapping."""
    cap = cap or max(1, comm.get_option("trace_events"))
    buf = np.zeros(cap, dtype=_REC)
    n = C.c_int64()
    check(lib().tl_trace_read(comm._h, buf.ctypes.data, cap, C.byref(n)), "tl_trace_read")
    out = []
    for r in buf[:n.value]:
        kind = KINDS[int(r["kind"])]
        if kind == "sm_clock" and not clocks:   # SM cycle stamps (t_ns holds clock64), diagnostics only
            continue
        ev = {"rank": int(r["rank"]), "unit": UNITS[int(r["unit"])], "kind": kind,
              "tile": int(r["tile"]) & 0xFFFFFF, "channel": None, "t_ns": int(r["t_ns"])}
        if kind in ("copy_start", "copy_end", "notify"):
            ev["peer"] = int(r["tile"]) >> 24
        out.append(ev)
    out.sort(key=lambda e: e["t_ns"])
    return out


def to_jsonl(events, path: str):
    with open(path, "w") as f:
        for e in events:
            f.write(json.dumps(e) + "\n")


def _intervals_union(iv):
    """Total length of the union of [a, b) intervals."""
    tot, end = 0, None
    for a, b in sorted(iv):
        if end is None or a > end:
            tot += b - a
            end = b
        elif b > end:
            tot += b - end
            end = b
    return tot


def _intersect_len(iv1, iv2):
    """Length of (union of iv1) intersected with (union of iv2)."""
    def merge(iv):
        out = []
        for a, b in sorted(iv):
            if out and a <= out[-1][1]:
                out[-1][1] = max(out[-1][1], b)
            else:
                out.append([a, b])
        return out
    A, B = merge(iv1), merge(iv2)
    i = j = tot = 0
    while i < len(A) and j < len(B):
        lo, hi = max(A[i][0], B[j][0]), min(A[i][1], B[j][1])
        if hi > lo:
            tot += hi - lo
        if A[i][1] < B[j][1]:
            i += 1
        else:
            j += 1
    return tot


def analyze_trace(events):
    """SPEC analyze_trace: per (rank, unit) busy time (union of tile / copy spans) and wait time
    (sum of wait spans), spans paired by (rank, unit, tile[, peer]); unmatched starts / ends are
    reported as diagnostics.  Also, per rank, the time its copy spans overlap its compute spans."""
    opens, spans, waits, diag = {}, {}, {}, []
    pair = {"tile_start": ("tile_end", spans), "copy_start": ("copy_end", spans), "wait_start": ("wait_end", waits)}
    closers = {v[0]: k for k, v in pair.items()}
    notifies = {}
    for e in events:
        key = (e["rank"], e["unit"], e.get("tile"), e.get("peer"))
        if e["kind"] in pair:
            if (e["kind"],) + key in opens:
                diag.append(f"duplicate {e['kind']} {key}")
            opens[(e["kind"],) + key] = e["t_ns"]
        elif e["kind"] in closers:
            start = closers[e["kind"]]
            t0 = opens.pop((start,) + key, None)
            if t0 is None:
                diag.append(f"{e['kind']} without {start}: {key}")
                continue
            store = pair[start][1]
            store.setdefault((e["rank"], e["unit"]), []).append((t0, e["t_ns"]))
        elif e["kind"] == "notify":
            notifies[(e["rank"], e["unit"])] = notifies.get((e["rank"], e["unit"]), 0) + 1
    for k in opens:
        diag.append(f"{k[0]} without end: {k[1:]}")
    units = sorted(set(spans) | set(waits) | set(notifies))
    per = {}
    for ru in units:
        per[f"{ru[0]}/{ru[1]}"] = {"busy_ns": _intervals_union(spans.get(ru, [])),
                                   "wait_ns": sum(b - a for a, b in waits.get(ru, [])),
                                   "wait_pairs": len(waits.get(ru, [])), "notifies": notifies.get(ru, 0),
                                   "spans": len(spans.get(ru, []))}
    overlap = {}
    for r in sorted({ru[0] for ru in units}):
        cp, cm = spans.get((r, "copy"), []), spans.get((r, "compute"), [])
        if cp:
            overlap[r] = {"copy_ns": _intervals_union(cp), "copy_under_compute_ns": _intersect_len(cp, cm)}
    t = [e["t_ns"] for e in events]
    return {"per_unit": per, "overlap": overlap, "diagnostics": diag,
            "span_ns": (max(t) - min(t)) if t else 0}
