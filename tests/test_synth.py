"""Generator self-checks (SURVEY.md App. B vectors; BASELINE.json configs)."""
import numpy as np

import synth


def test_splitmix_vector():
    z = synth.mix(np.array([synth.stream_id(3, 3, 0) + int(synth.GAMMA)], dtype=np.uint64))
    assert int(z[0]) == 0xF0E06EAEF05DE1F0


def test_u01_draws():
    exp = {
        (3, 3, 0): [0.9409245659920695, 0.4999259600429915, 0.24909005659599848],
        (3, 4, 0): [0.7295201338257296, 0.6579982467357524, 0.15026196501388522],
        (5, 3, 0): [0.6103650841670083, 0.5041729682725296, 0.9461376936637548],
        (2, 4, 0): [0.8504979468379756, 0.9265437292823202, 0.011775397096635554],
    }
    for s, v in exp.items():
        assert synth.u01(synth.stream_id(*s), 0, 3).tolist() == v


def test_config3_x_dc():
    x = synth.density(3, 4)
    dc = synth.sensitivity(3, x)
    assert x[0] == 0.9409836414260775
    assert dc[0] == -3.266036594742885


def test_config4_ground_structure():
    c, holes = synth.ground_structure(4)
    assert c.shape == (1385707, 2)
    assert c[0, 0] == 0.770235014120229 and c[0, 1] == 0.5216003802405329
    np.testing.assert_allclose(holes[0], [1850.63, 326.78, 85.83], atol=0.01)
    assert not np.any((c[:, 0] >= 1000) & (c[:, 1] >= 500))


def test_config_sizes():
    assert synth.centroids(1).shape == (1200, 2)
    assert synth.centroids(2).shape == (60000, 2)
    c3 = synth.centroids(3)
    assert c3.shape == (1024000, 3) and c3[1].tolist() == [1.5, 0.5, 0.5]
    k = synth.kuhn_tets(2, 2, 2)
    assert k.shape == (48, 3)
    # Kuhn centroids are quarters (exact)
    assert np.all(k * 4 == np.round(k * 4))


def test_sample_rows_distinct():
    r = synth.sample_rows(5, 12_000_000, 1000)
    assert len(set(r.tolist())) == 1000 and r.min() >= 0 and r.max() < 12_000_000
