"""InfluenceMaximizer / as_graph on the device vs the reference
(tests/golden/est_cases.npz, make_golden_estimator.py)."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def test_as_graph_matches_reference(gpu):
    from paper_2008_03095_b200.estimator import as_graph
    z = load_golden("est_cases")
    g = as_graph(z["arr"])
    for a, b in (("xadj", "xadj"), ("adj", "adj"), ("weights", "weights"), ("orig_ids", "orig")):
        assert np.array_equal(getattr(g, a), z[b])
    g2 = as_graph(z["arr"][:, :2].astype(np.int64))
    for a, b in (("xadj", "xadj2"), ("adj", "adj2"), ("weights", "weights2"), ("orig_ids", "orig2")):
        assert np.array_equal(getattr(g2, a), z[b])


@pytest.mark.parametrize("case", ["const", "file", "wc"])
def test_estimator_fit_score_match_reference(gpu, case):
    from paper_2008_03095_b200.estimator import InfluenceMaximizer
    z = load_golden("est_cases")
    X = z["arr"] if str(z[f"{case}_scheme"]) == "file" else z["arr"][:, :2].astype(np.int64)
    m = InfluenceMaximizer(k=int(z[f"{case}_k"]), num_simulations=int(z[f"{case}_r"]),
                           weight_scheme=str(z[f"{case}_scheme"]), random_state=int(z[f"{case}_seed"])).fit(X)
    assert np.array_equal(m.seeds_, z[f"{case}_seeds"])
    assert np.array_equal(m.seed_indices_, z[f"{case}_idx"])
    assert m.predict() is m.seeds_
    assert m.expected_spread_ == float(z[f"{case}_spread"])
    assert m.expected_spread_se_ == pytest.approx(float(z[f"{case}_se"]), rel=1e-12)
    assert m.score(r_eval=3000) == float(z[f"{case}_score"])


def test_estimator_validation(gpu):
    from paper_2008_03095_b200.estimator import InfluenceMaximizer
    with pytest.raises(AttributeError):
        InfluenceMaximizer().predict()
    with pytest.raises(ValueError):
        InfluenceMaximizer(k=1).fit(np.zeros((0, 2)))
    with pytest.raises(ValueError):
        InfluenceMaximizer(k=1).fit([(3, 3), (4, 4)])
    with pytest.raises(gpu.ConstraintError):
        InfluenceMaximizer(k=5).fit([(0, 1), (1, 2)])
    with pytest.raises(gpu.ConstraintError):
        InfluenceMaximizer(k=1, num_simulations=0).fit([(0, 1)])
    m = InfluenceMaximizer(k=2, weight_scheme="const:1.0").fit([(0, 1), (1, 2), (10, 11)])
    assert m.seeds_.tolist() == [0, 10]     # the reference docstring example
