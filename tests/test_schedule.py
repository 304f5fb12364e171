"""The online training schedule (reading R34), host logic.

Pinned to the rules the paper states: iterations double the sample count (Mueller 17);
training stops as soon as 30 % of the budget is used; after an iteration a new round
starts only if less than half of the training budget is used, otherwise the current
iteration continues until rendering starts; the rest of the budget renders."""
import pytest

from paper_2311_12818_b200 import mpg


@pytest.mark.parametrize("B", list(range(1, 64)) + [100, 256, 1000, 4096, 12345])
def test_schedule_follows_the_paper(B):
    iters, render = mpg.training_schedule(B)
    T = int(0.3 * B)
    assert sum(iters) == T and render == B - T                      # 30 % training, never splatted
    for j, n in enumerate(iters[:-1]):
        assert n == 1 << j                                          # doubling
        assert 2 * sum(iters[:j + 1]) < T                           # a new round only below half
    if iters:
        j = len(iters) - 1
        before = sum(iters[:-1])
        if iters[-1] != 1 << j:
            # the last round was cut at the training budget, or continued past half of it
            assert iters[-1] == T - before
            assert before + (1 << j) >= T or 2 * (before + (1 << j)) >= T


def test_schedule_examples():
    assert mpg.training_schedule(100) == ([1, 2, 4, 23], 70)
    assert mpg.training_schedule(10) == ([1, 2], 7)
    assert mpg.training_schedule(3) == ([], 3)
    assert mpg.training_schedule(100, 0.0) == ([], 100)
