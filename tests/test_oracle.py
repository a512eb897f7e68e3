"""The oracle itself, pinned before it is trusted (CPU only).

* against the golden fixtures generated from the UNMODIFIED reference
  (tests/golden/gen_golden.py, oracle/_ref) -- norms, clip scales, clip
  counts, noise-free clipped sums, a full fp32 reference step;
* against the reference test-suite's known answers (proj/tests/*.cpp);
* against the live compiled reference when oracle/_ref is present.
"""
import hashlib
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

FIXTURES = {
    "logreg": (lambda O: O.build_desc(O.LOGREG)),
    "fcnn": (lambda O: O.build_desc(O.FCNN)),
    "fcnn_104_50_2": (lambda O: O.custom_desc(O.FCNN, [(0, 104, 50, 0, 1, 0), (6, 0, 0, 0, 1, 0),
                                                       (0, 50, 2, 0, 1, 0)], (104,), 2)),
    "mnist_cnn": (lambda O: O.build_desc(O.MNIST_CNN)),
    "cifar_cnn": (lambda O: O.build_desc(O.CIFAR_CNN)),
    "embed_small": (lambda O: O.build_desc(O.EMBED, seq_len=16, vocab=50, hidden=8)),
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


@pytest.mark.parametrize("name", list(FIXTURES))
def test_restatement_matches_reference_fixtures(O, name):
    g = load(name)
    d = FIXTURES[name](O)
    B, C = int(g["B"]), float(g["clip"])
    assert list(g["blocks"]) == d.blocks
    # bit-exact init and synthetic data (models.cpp:359-375, dataset.cpp:126-237)
    assert sha(O.init_params(d, 0, np.float32)) == str(g["init_sha"])
    x32, y32 = O.synth(d, B, 0, np.float32)
    assert sha(x32) == str(g["x_sha"]) and sha(y32) == str(g["y_sha"])
    p64 = O.init_params(d, 0)
    np.testing.assert_array_equal(p64[:64], g["init64_head"])
    x, y = O.synth(d, B, 0)
    _, norms, nclip, cs = O.dpsgd_step(d, x, y, p64, C, 0.0, 0.1, 1, 0, 0)
    np.testing.assert_allclose(norms, g["norms"], rtol=1e-12)
    assert nclip == int(g["clipped_count"])
    want = g["clipped_sum"]
    got = cs[:: int(g["every"])]
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


def test_mnist_fp32_step_is_reproduced_bitwise(O):
    """The fp32 views-path tail over the reference's own fp32 stacks equals
    one reference fp32 dpsgd_step bit for bit (dpsgd.cpp:232-322)."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    g = load("mnist_cnn")
    d = O.build_desc(O.MNIST_CNN)
    B = int(g["B"])
    p32 = O.init_params(d, 0, np.float32)
    x, y = O.synth(d, B, 0, np.float32)
    R = O.RefModel(d, O.GROUPCONV, B, p32, np.float32)
    stacks, _ = R.per_example(x, y)
    newp, norms, nclip = O.aggregate_f32(d.blocks, stacks, p32, 1.0, 1.1, 0.1, 0, 0, B)
    np.testing.assert_array_equal(newp, g["step_params_f32"])
    np.testing.assert_array_equal(norms, g["step_norms_f32"])
    assert nclip == int(g["step_clipped"])


def test_noise_matches_reference(O):
    g = load("rng")
    assert O.port().orc_rng_value_at(0, 1 << 32, 0) == int(g["rng_value_at_0"][0])
    assert O.port().orc_rng_value_at(0, 1 << 32, 1) == int(g["rng_value_at_0"][1])
    np.testing.assert_array_equal(O.gaussian(0, 1 << 32, 1001), g["gauss_f64"])
    np.testing.assert_array_equal(O.gaussian(0, 1 << 32, 1001, np.float32), g["gauss_f32"])
    np.testing.assert_array_equal(O.gaussian(99, 7, 7, np.float32), g["gauss_f32_odd"])
    m = load("mnist_cnn")
    d = O.build_desc(O.MNIST_CNN)
    noise = np.concatenate([O.gaussian(0, O.noise_stream(0, p), n, np.float32)
                            for p, n in enumerate(d.blocks)])
    np.testing.assert_array_equal(noise, m["noise_f32"])
    # SURVEY 8(c) anchors
    np.testing.assert_allclose(noise[:4], [-1.36026716, -0.282528609, -0.736619234, -0.701791048],
                               rtol=1e-7)


def test_parameter_counts(O):
    """proj/tests/test_models.cpp:26-35."""
    assert O.build_desc(O.LOGREG).param_count == 105
    assert O.build_desc(O.FCNN).param_count == 5760
    assert O.build_desc(O.MNIST_CNN).param_count == 26010
    assert O.build_desc(O.CIFAR_CNN).param_count == 605226
    assert O.build_desc(O.EMBED).param_count == 160098
    assert O.build_desc(O.LSTM_MODEL).param_count == 1081002
    assert O.build_desc(O.EMBED, hidden=100).param_count == 1000602


def test_clip_kats(O):
    """proj/tests/test_dpsgd.cpp:37-47, 77-82: (6,8) at C=5 -> (3,4); norm == C
    is left alone; zero gradients have scale 1."""
    # one unit, sigma 0, lr 1: the update is exactly -clip(g)
    p, norms, n = O.aggregate_f32([2], np.array([6.0, 8.0], np.float32),
                                  np.zeros(2, np.float32), 5.0, 0.0, 1.0, 0, 0, 1)
    np.testing.assert_array_equal(-p, [3.0, 4.0])
    assert n == 1 and norms[0] == 10.0
    p, _, n = O.aggregate_f32([2], np.array([3.0, 4.0], np.float32), np.zeros(2, np.float32),
                              5.0, 0.0, 1.0, 0, 0, 1)
    np.testing.assert_array_equal(-p, [3.0, 4.0])
    assert n == 0
    p, norms, n = O.aggregate_f32([2], np.zeros(2, np.float32), np.zeros(2, np.float32), 5.0,
                                  0.0, 1.0, 0, 0, 1)
    assert n == 0 and norms[0] == 0 and np.all(p == 0)


def test_outer_product_kat(O):
    """proj/tests/test_strategies.cpp:112-131: a=(1,2), d=(3,4) -> [[3,6],[4,8]]
    as the (in,out) per-example dW of a linear layer with no bias effect."""
    d = O.custom_desc(O.LOGREG, [(0, 2, 2, 0, 1, 0)], (2,), 2)
    # choose W so that dlogits = onehot-softmax is irrelevant: check the rule
    # dW_i = a_i (x) delta_i directly through the restatement's per-example grads
    x = np.array([[1.0, 2.0]])
    y = np.array([0.0])
    W = np.zeros(d.param_count)
    st, _, _ = O.per_example_grads(d, x, y, W)
    delta = st[4:6]  # bias block = delta
    np.testing.assert_allclose(st[:4].reshape(2, 2), np.outer(x[0], delta))


def test_sigma0_loose_clip_equals_sgd(O):
    """proj/tests/test_dpsgd.cpp:204-226."""
    d = O.build_desc(O.FCNN)
    p = O.init_params(d, 11)
    x, y = O.synth(d, 8, 3)
    a, _, nclip, _ = O.dpsgd_step(d, x, y, p, 1e6, 0.0, 0.5, 1, 0, 0)
    b = O.sgd_step(d, x, y, p, 0.5)
    assert nclip == 0
    np.testing.assert_allclose(a, b, rtol=1e-9, atol=1e-12)


def test_microbatch_m_equals_b(O):
    """proj/tests/test_dpsgd.cpp:294-338: m = B is clip(mean grad) + noise."""
    d = O.build_desc(O.FCNN)
    p = O.init_params(d, 7)
    x, y = O.synth(d, 4, 0)
    got, norms, _, cs = O.dpsgd_step(d, x, y, p, 0.25, 0.5, 0.2, 4, 50, 3)
    st, _, _ = O.per_example_grads(d, x, y, p)
    mean = np.concatenate([blk.mean(axis=0) for blk in O.split_stacks(d, st, 4)])
    n = np.linalg.norm(mean)
    clipped = mean * min(1.0, 0.25 / n)
    noise = np.concatenate([O.gaussian(50, O.noise_stream(3, q), k)
                            for q, k in enumerate(d.blocks)])
    want = p - 0.2 * (clipped + 0.5 * 0.25 * noise)
    assert abs(norms[0] - n) <= 1e-12 * n
    np.testing.assert_allclose(got, want, rtol=1e-10, atol=1e-13)


def test_noise_variance(O):
    """proj/tests/test_dpsgd.cpp:135-153: variance within 2% of (sigma C / B)^2."""
    draws = np.concatenate([O.gaussian(1234, O.noise_stream(t, 0), 2) for t in range(50000)])
    want = 1.0
    assert abs(draws.var() - want) < 0.02 * want


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__))), "oracle", "_ref", "libpegrad_ref.so")), reason="no oracle/_ref")
@pytest.mark.parametrize("kind,kw,B,strat,m", [(0, {}, 8, 2, 1), (1, {}, 8, 5, 2),
                                               (1, {}, 8, 3, 1),  # norms: the two-pass step
                                               (2, {}, 4, 4, 1), (2, {}, 4, 1, 2),
                                               (4, dict(seq_len=8, vocab=20, hidden=4), 4, 5, 1)])
def test_restatement_matches_live_reference(O, kind, kw, B, strat, m):
    d = O.build_desc(kind, **kw)
    p = O.init_params(d, 3)
    x, y = O.synth(d, B, 5)
    R = O.RefModel(d, strat, B, p)
    rs, rn = R.per_example(x, y, want_stacks=strat != O.NORMS)
    st, nsq, _ = O.per_example_grads(d, x, y, p)
    if rs is not None:
        assert np.abs(st - rs).max() <= 1e-12 * max(1.0, np.abs(rs).max())
    np.testing.assert_allclose(np.sqrt(nsq), rn, rtol=1e-12)
    for step in range(3):
        got, norms, nclip, _ = O.dpsgd_step(d, x, y, p, 0.5, 0.7, 0.1, m, 9, step)
        rn, rclip = R.step(x, y, 0.5, 0.7, 0.1, m, 9, step)
        np.testing.assert_allclose(norms, rn, rtol=1e-12)
        assert nclip == rclip
        np.testing.assert_allclose(got, R.params(), rtol=1e-12, atol=1e-15)
        p = got


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__))), "oracle", "_ref", "libpegrad_ref.so")), reason="no oracle/_ref")
@pytest.mark.parametrize("kind,strat", [(1, 3), (1, 2), (2, 4)])
def test_weighted_grad_sum_matches_restatement(O, kind, strat):
    """GradEngine::weighted_grad_sum (strategies.cpp:432-450, one weighted
    backward) equals sum_i w_i g_i over the restatement's per-example stacks:
    the identity the norms-only two-pass step (dpsgd.cpp:194-230) rests on."""
    d = O.build_desc(kind)
    B = 6
    p = O.init_params(d, 2)
    x, y = O.synth(d, B, 4)
    w = np.random.default_rng(0).uniform(0.1, 1.0, B)
    R = O.RefModel(d, strat, B, p)
    got = R.weighted_grad_sum(x, y, w)
    st, _, _ = O.per_example_grads(d, x, y, p)
    want = np.concatenate([(w[:, None] * b).sum(0) for b in O.split_stacks(d, st, B)])
    np.testing.assert_allclose(got, want, rtol=1e-10, atol=1e-13 * np.abs(want).max())
