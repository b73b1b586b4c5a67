"""The three-party ledger (transport.py: the reference's CommStats accounting), no GPU."""


def test_ledger_ring_fast_path_equals_round():
    """Ledger.ring (the eager path's per-call charge, no per-send checks)
    charges exactly what round() with the three ring sends does, and records
    the same sends under a graph capture."""
    from paper_2104_10949_b200.transport import Ledger

    a, b = Ledger(), Ledger()
    for label, words in [("mul", 7), ("and", 0), ("open", 1 << 20), ("mul", 3)]:
        a.ring(label, words)
        b.round(label, [(i, (i + 1) % 3, words) for i in range(3)])
    for ta, tb in zip(a.parties, b.parties):
        assert ta.stats.__dict__ == tb.stats.__dict__
    with a.capture() as ca:
        a.ring("x", 5)
    with b.capture() as cb:
        b.round("x", [(i, (i + 1) % 3, 5) for i in range(3)])
    assert [s.__dict__ for s in ca.charge] == [s.__dict__ for s in cb.charge]
    a.enabled = False
    a.ring("off", 1)
    assert a.parties[0].stats.rounds == 4
