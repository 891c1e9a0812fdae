"""Host-side scheduling rules of the batched solver (no GPU needed).

``krylov.concurrent_groups`` splits a small solve into concurrently run sub-batches; per-mode
results never depend on it (batch invariance), so it may depend on the batch size, while the
native pass segmentation may not (a rule on the system only, DESIGN.md §4/§7).
"""

import pytest

from paper_2009_06725_b200.krylov import concurrent_groups


def test_groups_rule(monkeypatch):
    monkeypatch.delenv("SS_CONCURRENT_GROUPS", raising=False)
    monkeypatch.delenv("SS_FUSED", raising=False)
    assert concurrent_groups(32_937_682, 1) == 1          # large systems: one batch
    assert concurrent_groups(500_000, 17) == 1
    assert concurrent_groups(9_103, 9) == 3               # config 1: 3 groups of 3
    assert concurrent_groups(8_782, 17) == 4              # pipe3d: at most 4
    assert concurrent_groups(9_103, 2) == 1               # groups of >= 3 modes
    assert concurrent_groups(7_033, 128) == 4


@pytest.mark.parametrize("value,expect", [("2", 2), ("1", 1), ("64", 9)])
def test_groups_override(monkeypatch, value, expect):
    monkeypatch.delenv("SS_FUSED", raising=False)
    monkeypatch.setenv("SS_CONCURRENT_GROUPS", value)
    assert concurrent_groups(9_103, 9) == expect          # capped at the batch size


def test_fused_tick_runs_one_group(monkeypatch):
    """The fused tick is a cooperative launch over every SM: never two at once."""
    monkeypatch.delenv("SS_CONCURRENT_GROUPS", raising=False)
    monkeypatch.setenv("SS_FUSED", "1")
    assert concurrent_groups(9_103, 9) == 1
    monkeypatch.setenv("SS_FUSED", "0")
    assert concurrent_groups(9_103, 9) == 3
