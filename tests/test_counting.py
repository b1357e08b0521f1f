"""Multiply accounting (counting.py:12-52 of the reference): the counter and
context-manager semantics, and the reference's linear-cost acceptance
criterion (test_acceptance.py: test_criterion_5_linear_cost_scaling) on the
per-sample counts of the kernels' formulation."""

import numpy as np
import pytest

from paper_2204_07104_b200 import counting
from paper_2204_07104_b200.counting import count_multiplies, counter, epoch_multiplies, factor_sample_multiplies


def test_counter_off_by_default_and_nested_blocks():
    counter.add(5)
    assert not counter.enabled
    with count_multiplies() as outer:
        counter.add(3)
        with count_multiplies() as inner:
            counter.add(4)
        assert inner.total == 4 and outer.so_far == 7
    assert outer.total == 7 and not counter.enabled


def test_linear_cost_scaling_criterion():
    # the reference's criterion: doubling r_core at fixed J within 2.4x,
    # log-log slope over J in {4, 8, 16} at most 1.2 (order 3)
    ratio_r = factor_sample_multiplies((8, 8, 8), 8) / factor_sample_multiplies((8, 8, 8), 4)
    costs = [factor_sample_multiplies((j, j, j), 4) for j in (4, 8, 16)]
    slope = float(np.polyfit(np.log([4, 8, 16]), np.log(costs), 1)[0])
    assert ratio_r <= 2.4 and slope <= 1.2


@pytest.mark.gpu
def test_train_reports_its_multiplies():
    from paper_2204_07104_b200 import ModelConfig, TrainConfig, generate_synthetic, init_model, split, train

    t, _ = generate_synthetic((30, 32, 34), 3000, (4, 4, 4), 4, noise_sigma=0.1, seed=3)
    ds = split(t, 0.1, seed=3)
    m = init_model(t.dims, ModelConfig((4, 4, 4), 4, 0.5, seed=1))
    cfg = TrainConfig(epochs=3, seed=1, core_batch_cap=1000)
    with count_multiplies() as c:
        train(m, ds, cfg)
    assert c.total == 3 * epoch_multiplies((4, 4, 4), 4, ds.train.nnz, 1000)
    assert counting.counter.enabled is False
