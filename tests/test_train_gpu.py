"""bench::train and bench::run_bench (proj/core/src/harness.cpp:85-167,319-382)
through the Python mirror, pinned to the UNMODIFIED compiled reference
(oracle/_ref, bench::train<float>) on the same data, seeds and DP settings:

* the per-epoch example order (RngState(seed, 2^40 + epoch) Fisher-Yates),
  by the library's pgb_shuffle_order, equals a Python restatement (CPU test);
* train: final parameters (per-block normwise rel 1e-4 after the run's
  steps of fp32 drift), per-epoch mean evaluation losses (rel 1e-4), final
  train accuracy (equal up to one example at a near-tie logit), step count;
* run_bench: a BenchRecord per batch size with positive epoch times.
"""
import numpy as np
import pytest


def test_shuffle_order_matches_restatement(P):
    from paper_2010_09063_b200.harness import _shuffle, _shuffle_py
    for n, seed in [(1, 0), (2, 3), (97, 0), (1000, 7)]:
        a = np.arange(n, dtype=np.int64)
        b = np.arange(n, dtype=np.int64)
        for epoch in range(3):  # passes compose: each epoch reshuffles the last
            _shuffle(a, seed, epoch)
            _shuffle_py(b, seed, epoch)
            np.testing.assert_array_equal(a, b)
            assert sorted(a.tolist()) == list(range(n))


CASES = [
    # name, kind, strategy (ours / reference), n, batch, epochs, private, sigma
    ("fcnn_dp", 1, 1, 256, 32, 2, True, 1.1),
    ("logreg_dp", 0, 2, 200, 40, 2, True, 1.1),
    ("fcnn_sgd", 1, 1, 128, 32, 1, False, 0.0),
    ("mnist_dp", 2, 4, 64, 16, 1, True, 1.1),
]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_train_matches_compiled_reference(P, O, case):
    if not O.ref_available():
        pytest.skip("compiled reference not built")
    name, kind, strat, n, batch, epochs, private, sigma = case
    desc = P.build_desc(P.ModelKind(kind))
    od = O.build_desc(kind)
    model = P.build_from_desc(desc, 0)
    p0 = model.flat_params()
    data = P.synth_for_model(desc, n, 3)
    cfg = P.DpConfig(clip_norm=1.0, noise_multiplier=sigma, learning_rate=0.1, seed=5)
    res = P.train(model, data, P.Strategy(strat), P.ExecMode.graph, cfg, batch, epochs, private)
    want_p, want_l, want_acc, want_steps = O.ref_train(
        od, p0, data.inputs, data.labels, strat, 1.0, sigma, 0.1, 1, 5, batch, epochs, private)
    assert res.steps == want_steps == epochs * (n // batch)
    got = model.flat_params().astype(np.float64)
    off = 0
    for blk in od.blocks:
        g, w = got[off:off + blk], want_p[off:off + blk].astype(np.float64)
        assert np.linalg.norm(g - w) <= 1e-4 * np.linalg.norm(w), (name, off)
        off += blk
    np.testing.assert_allclose(res.epoch_mean_loss, want_l, rtol=1e-4)
    assert abs(res.final_train_accuracy - want_acc) <= 1.0 / n + 1e-12


@pytest.mark.gpu
def test_run_bench_records(P):
    desc = P.build_desc(P.ModelKind.fcnn)
    data = P.synth_for_model(desc, 512, 0)
    opts = P.RunOptions(batch_sizes=[32, 128, 1024], epochs=2, clip_norm=1.0,
                        noise_multiplier=1.1, learning_rate=0.1, seed=0)
    recs = P.run_bench(P.ModelKind.fcnn, data, P.Strategy.vmap, opts)
    assert [r.batch_size for r in recs] == [32, 128, 1024]
    assert recs[2].status == "skip"  # batch larger than the dataset (harness.cpp:120-127)
    for r in recs[:2]:
        assert r.status == "ok" and len(r.epoch_seconds) == 2 and r.median_epoch_seconds > 0
