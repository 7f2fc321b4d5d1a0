"""The executor's early-stop rule against the reference's own detect_stop
(progress.cpp:90-124, compiled in place into oracle/_ref): identical stop
iteration and cause on random loss / accuracy streams with NaN/inf losses,
accuracy ties and plateaus, and patience 0..4 (CPU)."""
import math
import random

import pytest

from oracle import ref
from paper_2312_02515_b200.executor import detect_stop

pytestmark = pytest.mark.skipif(not (ref.available() or ref.build()),
                                reason="oracle/_ref not built (needs /root/reference)")


def _stream(rng):
    n = rng.randint(0, 12)
    losses = [rng.choice([0.5, 1.0, 2.0, float("nan"), float("inf"), -float("inf")])
              if rng.random() < 0.15 else rng.uniform(0, 3) for _ in range(n)]
    m = rng.randint(0, 12)
    accs = [rng.choice([0.1, 0.2, 0.3, 0.4, 0.5]) for _ in range(m)]
    return losses, accs


def test_detect_stop_matches_reference():
    rng = random.Random(2312)
    fired = {"nan_loss": 0, "accuracy_decline": 0, None: 0}
    for _ in range(3000):
        losses, accs = _stream(rng)
        patience = rng.randint(0, 4)
        ours = detect_stop(losses, accs, patience)
        assert ours == ref.detect_stop(losses, accs, patience), (losses, accs, patience)
        fired[ours[1] if ours else None] += 1
    assert min(fired.values()) > 100  # every outcome exercised


def test_detect_stop_known_answers():
    nan = float("nan")
    assert detect_stop([1.0, nan, 2.0]) == (2, "nan_loss")
    assert detect_stop([1.0, 1.0], [0.5, 0.4, 0.4, 0.3], patience=3) == (4, "accuracy_decline")
    # tie on the iteration: the NaN stop wins (progress.cpp:120-122)
    assert detect_stop([1, 1, 1, nan], [0.5, 0.4, 0.4, 0.3], patience=3) == (4, "nan_loss")
    assert detect_stop([1.0, 2.0], [0.1, 0.2, 0.3]) is None
    assert detect_stop([], [0.5, 0.4, 0.3, 0.2], patience=0) is None
    assert detect_stop([1.0, math.inf]) == (2, "nan_loss")
