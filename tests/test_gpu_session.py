"""Live session on the GPU (session.py:119-290 semantics): the virtual-clock replay with the device
positive pool, the GPU trainer and the GPU repository publishes the same lists at the same
ticks with the same counters as the reference's own run_simulated (golden), is bitwise
reproducible, and every publication verifies its CRC32."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def run(otf, golden):
    from paper_1407_4764_b200 import session as S

    repo = otf.Repository.dense(otf.FeatureStore(golden["sess_test_x"]))
    cfg = S.SessionConfig(rate=12.0, ranker=otf.RankerConfig(k=25, interval=0.18),
                          trainer=otf.TrainerConfig(lam=0.1, batch_size=16), steps_per_second=100.0)
    sess = S.QuerySession("s", "class_00", repo, golden["sess_neg"], cfg, trainer_seed=5)
    pubs = []
    S.run_simulated(sess, golden["sess_feed"], 2.0, on_publish=pubs.append)
    return sess, pubs


def test_replay_matches_reference_session(otf, golden):
    sess, pubs = run(otf, golden)
    assert len(pubs) == len(golden["sess_ids"])
    meta = np.array([[p.ranked.model_version, p.positives_fed, p.steps_applied, p.lists_published] for p in pubs])
    np.testing.assert_array_equal(meta, golden["sess_meta"])
    np.testing.assert_array_equal([p.ranked.produced_at for p in pubs], golden["sess_at"])
    for p, ref_ids in zip(pubs, golden["sess_ids"]):
        assert p.verify_checksum()
        assert list(p.ranked.ids) == list(ref_ids)
    np.testing.assert_allclose(sess.trainer.snapshot().weights, golden["sess_w"], rtol=1e-10, atol=1e-14)
    assert sess.state == "stopped"
    assert sess.stats()["lists_published"] == len(pubs)


def test_replay_is_bitwise_reproducible(otf, golden):
    _, a = run(otf, golden)
    _, b = run(otf, golden)
    assert [p.checksum for p in a] == [p.checksum for p in b]
