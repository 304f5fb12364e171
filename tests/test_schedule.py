"""The online training schedule (reading R34).

The library's schedule (mpg_training_schedule, C ABI, host code -- no GPU needed) equals
the oracle's pass-by-pass simulation of the paper's rules for every budget; the oracle is
pinned to the rules' consequences: iterations double the sample count (Mueller 17);
training stops as soon as 30 % of the budget is used; after an iteration a new round starts
only if less than half of the training budget is used, otherwise the current iteration
continues until rendering starts; the rest of the budget renders (never splats training)."""
import pytest

from oracle import oracle as O
from paper_2311_12818_b200 import mpg


@pytest.mark.parametrize("B", list(range(0, 64)) + [100, 256, 1000, 4096, 12345, 10 ** 6])
def test_oracle_schedule_follows_the_paper(B):
    iters, render = O.training_schedule(B)
    T = int(0.3 * B)
    assert sum(iters) == T and render == B - T                      # 30 % training, never splatted
    for j, n in enumerate(iters[:-1]):
        assert n == 1 << j                                          # doubling
        assert 2 * sum(iters[:j + 1]) < T                           # a new round only below half
    if iters:
        j = len(iters) - 1
        before = sum(iters[:-1])
        assert iters[-1] >= min(1 << j, T - before)                 # the last round is never cut short
        if iters[-1] > 1 << j:                                      # ... and extended only past half
            assert 2 * (before + (1 << j)) >= T


def test_library_schedule_equals_oracle():
    for B in list(range(0, 3000)) + [12345, 10 ** 6, 10 ** 9]:
        for f in (0.3, 0.0, 0.5, 1.0, 0.25):
            assert mpg.training_schedule(B, f) == O.training_schedule(B, f), (B, f)


def test_schedule_examples():
    assert mpg.training_schedule(100) == ([1, 2, 4, 23], 70)
    assert mpg.training_schedule(10) == ([1, 2], 7)
    assert mpg.training_schedule(3) == ([], 3)
    assert mpg.training_schedule(100, 0.0) == ([], 100)
