"""Item tables of the class-decomposed block stage (host logic, CPU only).

The library partitions a temporal block's (step, old slice) pairs into items
(stride, residue class, slice range, <= 8 step columns); the item coefficient
kernel gives entry (step, t) to every item whose range holds t, whose stride
equals the entry's weight and whose columns hold the step.  Every entry of
every schedule (oracle restatement of schedule.py:97-151) must therefore be
owned by exactly one item, and no item may claim a pair outside the schedules.
"""

import ctypes as C

import numpy as np
import pytest

from paper_1004_5128_b200 import _lib

CAP = 200


def item_table(kind, kb0, bt, ts, te, base, tblock, cols=8):
    L = _lib.load()
    out = (C.c_int64 * (20 * CAP))()
    n = C.c_int32(0)
    _lib.check(L.fg_block_item_table(kind, kb0, bt, ts, te, base, 0, tblock, cols, out, CAP, C.byref(n)))
    arr = np.frombuffer(out, dtype=np.int64).reshape(CAP, 20)
    return n.value, arr[: max(n.value, 0)]


def weight(segs, m):
    for m0, cnt, st in segs:
        d = m - m0
        if d < 0:
            return 0
        if d <= (cnt - 1) * st:
            return st if d % st == 0 else 0
    return 0


def check_ownership(kb0, bt, ts, te, base, tblock, cols=8):
    from oracle import fg_oracle as fo

    n, items = item_table(2, kb0, bt, ts, te, base, tblock, cols)
    if n < 0:
        return None
    segs = [fo.schedule_segments("adaptive", kb0 + b, base) for b in range(bt)]
    owned = {}
    for t_first, stride, n_sl, ncols, *steps in items.tolist():
        assert 1 <= ncols <= cols and stride >= 1 and n_sl >= 1
        assert ts <= t_first and t_first + (n_sl - 1) * stride < te
        for b in steps[:ncols]:
            for j in range(n_sl):
                t = t_first + j * stride
                if weight(segs[b], kb0 + b - t) == stride:
                    owned[(b, t)] = owned.get((b, t), 0) + 1
    want = set()
    for b in range(bt):
        offs, _w = fo.schedule("adaptive", kb0 + b, base)
        want |= {(b, kb0 + b - m) for m in offs.tolist() if ts <= kb0 + b - m < te}
    twice = {k: v for k, v in owned.items() if v != 1}
    assert not twice, f"kb0 {kb0} bt {bt} [{ts},{te}) a={base}: entries owned twice {sorted(twice)[:6]}"
    assert set(owned) == want, (f"kb0 {kb0} bt {bt} [{ts},{te}) a={base}: missing {sorted(want - set(owned))[:6]} "
                                f"extra {sorted(set(owned) - want)[:6]}")
    return n


@pytest.mark.parametrize("cols", [8, 16])
@pytest.mark.parametrize("base", [2, 3, 5, 8])
@pytest.mark.parametrize("tblock", [8, 16, 24, 32, 48, 64, 80, 128])
def test_every_entry_owned_once(base, tblock, cols):
    """Tails ([kb0 - tblock, kb0)) and main ranges ([0, kb0 - tblock)) of the
    first blocks (where the adaptive tail rule and the dense window share a
    class near t = 0) and of later blocks."""
    n_itemized = 0
    for kb0 in list(range(tblock, 12 * tblock + 1, tblock)) + [1000 // tblock * tblock, 2496 // tblock * tblock]:
        tb0 = max(0, kb0 - tblock)
        for ts, te in ((tb0, kb0), (0, tb0)):
            if te > ts and check_ownership(kb0, tblock, ts, te, base, tblock, cols) is not None:
                n_itemized += 1
    assert n_itemized > 0


def test_overlapping_groups_regression():
    """Block 16 of an a=5 run at tblock 16: the tail rule's entries near t = 0
    start a (stride 1, residue 0) group that the dense window of later steps
    grows into — the groups must be merged, not both kept."""
    assert check_ownership(16, 16, 0, 16, 5, 16) is not None


@pytest.mark.parametrize("cols", [8, 16])
def test_item_rows_bound_covers_blocks(cols):
    L = _lib.load()
    rows = C.c_int64(0)
    _lib.check(L.fg_block_item_rows(2, 1200, 48, 5, 0, cols, C.byref(rows)))
    worst = 0
    for kb0 in range(48, 1200, 48):
        bt = min(48, 1200 - kb0)
        tot = 0
        for ts, te in ((kb0 - 48, kb0), (0, kb0 - 48)):
            if te > ts:
                n, items = item_table(2, kb0, bt, ts, te, 5, 48, cols)
                tot += int(items[:, 2].sum()) if n > 0 else 0
        worst = max(worst, tot)
    assert rows.value == worst > 0
