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


def test_device_snapshot_publication_equals_host_snapshot(otf, golden):
    """OnlineTrainer.publish_to + Repository.rank_published (w copied trainer -> ranker on the
    device, CUDA event, no host round trip) rank exactly like rank(trainer.snapshot()), with the
    same version numbering; the trainer keeps its own buffer."""
    import pytest as _pytest

    repo = otf.Repository.dense(otf.FeatureStore(golden["sess_test_x"]))
    tr = otf.OnlineTrainer(repo.model_dim, golden["sess_neg"], otf.TrainerConfig(lam=0.1, batch_size=16, seed=2))
    with _pytest.raises(otf.NotReadyError):
        tr.publish_to(repo)
    tr.append_positives(golden["sess_feed"][:5])
    for _ in range(7):
        tr.step()
    it, ver = tr.publish_to(repo)
    a = repo.rank_published(tr, 25, produced_at=1.5, model_version=ver)
    snap = tr.snapshot()
    assert (snap.iteration, snap.version) == (it, ver)
    b = repo.rank(snap, 25, produced_at=1.5)
    assert list(a.ids) == list(b.ids) and np.array_equal(a.scores, b.scores)
    assert a.model_version == b.model_version == ver
    tr.step()  # a new iterate -> a new version; the published copy is unaffected until republished
    c = repo.rank_published(tr, 25, model_version=ver)
    assert list(c.ids) == list(a.ids)
    it2, ver2 = tr.publish_to(repo)
    assert (it2, ver2) == (it + 1, ver + 1)
    small = otf.Repository.dense(otf.FeatureStore(np.ones((10, 16), np.float32)))
    with _pytest.raises(otf.ConfigError):
        tr.publish_to(small)


def test_published_and_host_ranks_interleave_across_k(otf, golden):
    """rank_published (trainer-published device w) and host-memory rank share the repository's
    graph cache: interleaving them with k growing past the 8192-candidate layout and back must
    keep every list equal to the oracle-equivalent host rank of the same snapshot."""
    x = np.random.default_rng(11).standard_normal((20_000, golden["sess_test_x"].shape[1])).astype(np.float32)
    repo = otf.Repository.dense(otf.FeatureStore(x))
    tr = otf.OnlineTrainer(repo.model_dim, golden["sess_neg"], otf.TrainerConfig(lam=0.1, batch_size=16, seed=5))
    tr.append_positives(golden["sess_feed"][:5])
    n = repo.count
    for step, k in enumerate([10, 25, min(n, 9000), 10, min(n, 12_000), 3]):
        tr.step()
        _, ver = tr.publish_to(repo)
        snap = tr.snapshot()
        a = repo.rank_published(tr, k, model_version=ver)
        b = repo.rank(snap, k)
        assert list(a.ids) == list(b.ids) and np.array_equal(a.scores, b.scores), (step, k)
