"""Pin the oracle (oracle/xcmix_port.py) to the reference's golden fixtures.

The fixtures were produced by tests/golden/make_golden.py running the real
reference. Everything here is bit-exact: the oracle restates the same NumPy
arithmetic, so any difference means the oracle is not the reference.
Also re-states the reference's own known-answer tests for this path
(test_anns.py:30-33, :46-50; test_loss.py:72-76, :154-161).
"""

import numpy as np
import pytest

from conftest import golden
from oracle import xcmix_port as port


@pytest.mark.parametrize("name", ["step_c1_parity.npz", "step_dropout.npz"])
def test_step_matches_reference_bitwise(name):
    g = golden(name)
    L, wd = int(g["L"]), float(g["wd"])
    for t in range(int(g["n_steps"])):
        p = f"s{t}_"
        W = g[p + "W_before"].copy()
        emb = g[p + "emb"]
        keep = g[p + "keep"] if g[p + "keep"].size else None
        emb_used = emb * keep if keep is not None else emb
        loss, grad_emb, factors, uids = port.slate_step(
            W, emb_used, keep, g[p + "ids"], g[p + "y"], g[p + "origin"], g[p + "weights"],
            float(g[p + "lr"]), wd,
        )
        assert loss == float(g[p + "loss"])
        np.testing.assert_array_equal(grad_emb, g[p + "grad_emb"])
        np.testing.assert_array_equal(uids, g[p + "uids"])
        np.testing.assert_array_equal(W[uids], g[p + "W_after_touched"])
        untouched = np.ones(L, dtype=bool)
        untouched[uids] = False
        np.testing.assert_array_equal(W[untouched], g[p + "W_before"][untouched])


def test_step_fixture_exercises_row0_origin_quirk():
    g = golden("step_c1_parity.npz")
    # row 0 of batch 0 has fewer positives than k_p: its PAD slot code is
    # applied to every row (trainer.py:313)
    assert (g["s0_origin"][: int(g["k_p"])] == port.ORIGIN_PAD).any()


@pytest.mark.parametrize("name", ["slates_warm.npz", "slates_hard.npz"])
def test_slates_match_reference(name):
    g = golden(name)
    rng = np.random.default_rng(int(g["rng_seed"]))
    hard = g["hard"] if g["hard"].size else None
    k_r_eff = int(g["k_r"]) + (int(g["k_h"]) if hard is None else 0)
    ids, y, origin, weights = port.assemble_batch_slates(
        g["pos_padded"], g["n_pos"], g["batch_rows"], int(g["L"]), int(g["k_p"]), k_r_eff, rng, hard
    )
    np.testing.assert_array_equal(ids, g["ids"])
    np.testing.assert_array_equal(y, g["y"])
    np.testing.assert_array_equal(origin, g["origin"])
    np.testing.assert_array_equal(weights, g["weights"])


@pytest.mark.parametrize("name", ["refresh_random.npz", "refresh_ties.npz"])
def test_refresh_matches_reference(name):
    g = golden(name)
    ip, pid = g["pos_indptr"], g["pos_ids"]
    positives = [pid[ip[i] : ip[i + 1]] for i in range(len(ip) - 1)]
    ids = port.retrieve_hard_negatives(g["W"], g["E"], positives, int(g["k_h"]))
    np.testing.assert_array_equal(ids, g["ids"])


def test_update_matches_reference():
    g = golden("update.npz")
    W = g["W_before"].copy()
    port.apply_classifier_updates_arrays(W, g["ids"], g["grads"], float(g["lr"]), float(g["wd"]))
    np.testing.assert_array_equal(W, g["W_after"])


def test_update_rejects_nonfinite():
    W = np.zeros((3, 2), np.float32)
    with pytest.raises(port.OracleNumericalError):
        port.apply_classifier_updates_arrays(W, np.array([0]), np.array([[np.nan, 0.0]], np.float32), 0.1)
    assert not W.any()


def test_known_answer_tie_breaks():
    # test_anns.py:30-33 duplicate vectors -> [1, 2, 3]
    W = np.array([[0.0, 1.0], [1.0, 0.0], [1.0, 0.0], [0.5, 0.0]], dtype=np.float32)
    got = port.retrieve_hard_negatives(W, np.array([[1.0, 0.0]], np.float32), [np.zeros(0, np.int32)], 3)
    assert got[0].tolist() == [1, 2, 3]
    # test_anns.py:46-50 zero query -> lowest ids
    rng = np.random.default_rng(1)
    W = rng.standard_normal((20, 4)).astype(np.float32)
    got = port.retrieve_hard_negatives(W, np.zeros((1, 4), np.float32), [np.zeros(0, np.int32)], 5)
    assert got[0].tolist() == [0, 1, 2, 3, 4]


def test_known_answer_weights_and_factors():
    # test_loss.py:72-76 : (L - k_h)/k_r = 327.5575 at L=131073, k_h=50, k_r=400
    assert np.float32((131073 - 50) / 400) == np.float32(327.5575)
    # test_loss.py:154-161 : factors at s=0 are -0.5 / 0.5 / 0.5*(L-k_h)/k_r
    origin = np.array([port.ORIGIN_POS, port.ORIGIN_HARD, port.ORIGIN_RAND], np.int8)
    weights = np.array([1.0, 1.0, 9.0], np.float32)
    _, f = port.slate_factors(np.zeros((1, 3), np.float32), np.array([[1, 0, 0]], np.int8), origin, weights)
    assert f[0].tolist() == [-0.5, 0.5, 4.5]


def test_lr_schedule_known_answers():
    # test_trainer.py:38-47
    assert port.lr_at(0, 100, 10, 0.5) == 0.0
    assert port.lr_at(10, 100, 10, 0.5) == pytest.approx(0.5)
    assert port.lr_at(55, 100, 10, 0.5) == pytest.approx(0.25)
    assert port.lr_at(5, 100, 10, 1.0) == pytest.approx(0.5)
