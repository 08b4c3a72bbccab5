"""analyze_trace on hand-built traces: the host side of the device event trace.
CPU only."""
from paper_2503_20313_b200 import trace as T


def ev(rank, unit, kind, tile, t, peer=None):
    e = {"rank": rank, "unit": unit, "kind": kind, "tile": tile, "channel": None, "t_ns": t}
    if peer is not None:
        e["peer"] = peer
    return e


def test_empty_trace_is_all_zero():
    rep = T.analyze_trace([])
    assert rep["per_unit"] == {} and rep["diagnostics"] == [] and rep["span_ns"] == 0


def test_single_tile_span_busy_time():
    rep = T.analyze_trace([ev(0, "compute", "tile_start", 5, 100), ev(0, "compute", "tile_end", 5, 175)])
    assert rep["per_unit"]["0/compute"]["busy_ns"] == 75 and rep["diagnostics"] == []


def test_two_rank_ring_has_one_peer_wait_pair_per_rank():
    """a synthetic 2-rank ring trace -> R - 1 = 1 peer-wait pair per rank."""
    trace = []
    for r in (0, 1):
        trace += [ev(r, "compute", "tile_start", 0, 0), ev(r, "compute", "tile_end", 0, 50),
                  ev(r, "compute", "notify", 0, 55, peer=1 - r),
                  ev(r, "compute", "wait_start", 1, 60), ev(r, "compute", "wait_end", 1, 90),
                  ev(r, "compute", "tile_start", 1, 90), ev(r, "compute", "tile_end", 1, 140)]
    rep = T.analyze_trace(sorted(trace, key=lambda e: e["t_ns"]))
    for r in (0, 1):
        u = rep["per_unit"][f"{r}/compute"]
        assert u["wait_pairs"] == 1 and u["wait_ns"] == 30 and u["busy_ns"] == 100 and u["notifies"] == 1
    assert rep["diagnostics"] == []


def test_overlapping_spans_count_once_and_copy_overlap():
    trace = [ev(0, "compute", "tile_start", 0, 0), ev(0, "compute", "tile_start", 1, 10),
             ev(0, "compute", "tile_end", 0, 40), ev(0, "compute", "tile_end", 1, 60),
             ev(0, "copy", "copy_start", 3, 50, peer=1), ev(0, "copy", "copy_end", 3, 80, peer=1)]
    rep = T.analyze_trace(trace)
    assert rep["per_unit"]["0/compute"]["busy_ns"] == 60          # union of [0,40) and [10,60)
    assert rep["overlap"][0] == {"copy_ns": 30, "copy_under_compute_ns": 10}


def test_malformed_pairing_is_diagnosed():
    rep = T.analyze_trace([ev(0, "compute", "wait_end", 2, 5), ev(1, "copy", "copy_start", 0, 7, peer=0)])
    assert len(rep["diagnostics"]) == 2
