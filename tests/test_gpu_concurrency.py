"""Concurrency of the live path on the GPU: trainer and ranker threads (ctypes releases the GIL),
sessions sharing one repository, and calls on different CUDA streams sharing one handle.

Ports of the reference's own concurrency tests:
  * pkg/tests/test_trainer.py:215-242 — readers hammering snapshot() while the trainer steps see
    monotone versions and whole, bounded iterates (here the readers also publish the snapshot to
    the device and rank under it);
  * pkg/tests/test_session.py:225-244 / :246-264 — the wall-clock runner stops cleanly, and a
    reader polling latest_publication() at full speed never sees a torn publication (CRC32).
Plus the cases the GPU design adds: two sessions ticking concurrently on one repository (each list
is ranked under its own session's weights), device-mode and host-mode calls on different streams
of one handle (the handle orders them), and training steps overlapping ranking on the GPU.
"""

import threading
import time

import numpy as np
import pytest

import otf_oracle as O

pytestmark = pytest.mark.gpu


def clusters(dim, n_pos, n_neg, seed):
    rng = np.random.default_rng(seed)
    c = rng.standard_normal(dim)
    pos = (c + 0.3 * rng.standard_normal((n_pos, dim))).astype(np.float32)
    neg = rng.standard_normal((n_neg, dim)).astype(np.float32)
    pos /= np.linalg.norm(pos, axis=1, keepdims=True)
    neg /= np.linalg.norm(neg, axis=1, keepdims=True)
    return pos, neg


def test_concurrent_snapshots_and_publications_see_whole_iterates(otf):
    pos, neg = clusters(8, 50, 50, 9)
    x = np.random.default_rng(1).standard_normal((5000, 8)).astype(np.float32)
    repo = otf.Repository.dense(otf.FeatureStore(x))
    tr = otf.OnlineTrainer(8, neg, otf.TrainerConfig(lam=1.0, batch_size=8, seed=3))
    tr.step(pos)
    stop = threading.Event()
    failures: list[str] = []
    ranks = [0]

    def reader(publish):
        last_v = last_it = 0
        while not stop.is_set():
            if publish:
                it, v = tr.publish_to(repo)
                lst = repo.rank_published(tr, 20, model_version=v)
                if len(lst) != 20 or not np.all(np.diff(lst.scores) <= 0):
                    failures.append("bad published list")
                ranks[0] += 1
            else:
                snap = tr.snapshot()
                it, v = snap.iteration, snap.version
                if not np.all(np.isfinite(snap.weights)) or np.linalg.norm(snap.weights) > 1.0 + 1e-9:
                    failures.append("observed an out-of-range iterate")
            if v < last_v or it < last_it:
                failures.append("went backwards")
            last_v, last_it = v, it

    threads = [threading.Thread(target=reader, args=(i == 0,)) for i in range(3)]
    for t in threads:
        t.start()
    for _ in range(400):
        tr.step(pos)
    stop.set()
    for t in threads:
        t.join()
    assert failures == []
    assert ranks[0] > 0


def _session(otf, repo, neg, cfg, sid="s", seed=5):
    from paper_1407_4764_b200 import session as S

    return S.QuerySession(sid, "q", repo, neg, cfg, trainer_seed=seed)


def test_wall_runner_publishes_and_stops(otf):
    from paper_1407_4764_b200 import session as S

    pos, neg = clusters(16, 120, 150, 7)
    x = np.random.default_rng(2).standard_normal((3000, 16)).astype(np.float32)
    repo = otf.Repository.dense(otf.FeatureStore(x))
    cfg = S.SessionConfig(rate=60.0, ranker=otf.RankerConfig(k=20, interval=0.05),
                          trainer=otf.TrainerConfig(lam=0.02, batch_size=16), steps_per_second=200.0)
    sess = _session(otf, repo, neg, cfg)
    runner = S.WallRunner(sess, pos)
    runner.start()
    deadline = time.monotonic() + 5.0
    while sess.latest_publication() is None and time.monotonic() < deadline:
        time.sleep(0.01)
    pub = sess.latest_publication()
    assert pub is not None and pub.verify_checksum()
    runner.stop()
    assert runner.errors == []
    assert sess.state == S.STATE_STOPPED
    count = sess.stats()["lists_published"]
    time.sleep(0.15)
    assert sess.stats()["lists_published"] == count
    runner.stop()  # idempotent
    assert sess.state == S.STATE_STOPPED


def test_reads_are_never_torn_under_load(otf):
    """test_session.py:246-264 on the GPU path: 200 Hz feed, 500 steps/s, a rank every 10 ms, and a
    reader polling the latest publication as fast as it can."""
    from paper_1407_4764_b200 import session as S

    pos, neg = clusters(16, 400, 150, 8)
    x = np.random.default_rng(3).standard_normal((20_000, 16)).astype(np.float32)
    repo = otf.Repository.dense(otf.FeatureStore(x))
    cfg = S.SessionConfig(rate=200.0, ranker=otf.RankerConfig(k=25, interval=0.01),
                          trainer=otf.TrainerConfig(lam=0.02, batch_size=16), steps_per_second=500.0)
    sess = _session(otf, repo, neg, cfg)
    runner = S.WallRunner(sess, pos)
    runner.start()
    bad = polls = 0
    deadline = time.monotonic() + 0.8
    while time.monotonic() < deadline:
        pub = sess.latest_publication()
        polls += 1
        if pub is not None and not pub.verify_checksum():
            bad += 1
    runner.stop()
    assert runner.errors == []
    assert bad == 0
    st = sess.stats()
    assert st["lists_published"] > 0 and st["steps_applied"] > 0
    # every list was ranked exactly: descending scores, ids from the repository
    for p in sess.publication_history:
        assert p.verify_checksum()
        assert np.all(np.diff(p.ranked.scores) <= 0)


def test_two_sessions_share_one_repository(otf):
    """Two sessions (own trainers, own weights) tick concurrently on ONE repository: every list a
    session publishes equals rank(its own trainer's snapshot) — never the other session's w."""
    from paper_1407_4764_b200 import session as S

    x = np.random.default_rng(4).standard_normal((40_000, 32)).astype(np.float32)
    repo = otf.Repository.dense(otf.FeatureStore(x))
    cfg = S.SessionConfig(rate=0.0, ranker=otf.RankerConfig(k=50, interval=0.01),
                          trainer=otf.TrainerConfig(lam=0.05, batch_size=16), steps_per_second=100.0)
    failures: list[str] = []
    ticks = [0, 0]

    def drive(j):
        pos, neg = clusters(32, 30, 100, 100 + j)
        sess = _session(otf, repo, neg, cfg, sid=f"s{j}", seed=j)
        for v in pos:
            sess.feed_one(v)
        for it in range(60):
            for _ in range(1 + (it + j) % 3):
                sess.train_step()
            assert sess.rank_tick(float(it))
            pub = sess.latest_publication()
            host = repo.rank(sess.trainer.snapshot(), cfg.ranker.k)  # same iterate (this thread steps it)
            if not (np.array_equal(pub.ranked.ids, host.ids) and np.array_equal(pub.ranked.scores, host.scores)):
                failures.append(f"session {j} tick {it}: list ranked under another w")
            if pub.ranked.model_version != host.model_version:
                failures.append(f"session {j} tick {it}: version {pub.ranked.model_version} != {host.model_version}")
            ticks[j] += 1

    threads = [threading.Thread(target=drive, args=(j,)) for j in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert failures == []
    assert ticks == [60, 60]


def test_calls_on_different_streams_are_ordered(otf):
    """A device-mode rank on a side stream followed at once (no host sync) by host-mode ranks and
    scores on the handle's own stream, and device-mode ranks alternating between two streams: the
    handle orders every call after the previous one, so no call sees another's workspace."""
    import ctypes as C

    import torch

    from paper_1407_4764_b200 import _lib

    rng = np.random.default_rng(12)
    n, d, k = 300_000, 64, 500
    x = rng.standard_normal((n, d)).astype(np.float32)
    repo = otf.Repository.dense(otf.FeatureStore(x))
    W = rng.standard_normal((6, d))
    want = [O.top_k(O.score_dense(w, x), k)[0] for w in W]
    lib = _lib.load()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    Wd = torch.as_tensor(W, device="cuda")
    outs = [(torch.empty(k, dtype=torch.int64, device="cuda"), torch.empty(k, dtype=torch.float64, device="cuda"))
            for _ in W]
    got = C.c_int64()
    for rep in range(3):
        host = []
        for i in range(len(W)):
            st = (s1, s2)[i % 2]
            _lib.check(lib.otf_repo_rank(repo.handle, _lib.tptr(Wd[i]), k, _lib.tptr(outs[i][0]),
                                         _lib.tptr(outs[i][1]), None, C.byref(got), _lib.MEM_DEVICE,
                                         C.c_void_p(st.cuda_stream)))
            if i % 3 == 2:  # a host-mode call on the handle's own stream right behind it
                host.append((i, repo.rank(W[i], k).ids))
                sc = repo.score(W[i])
                assert np.max(np.abs(sc - O.score_dense(W[i], x))) <= 1e-6 * np.linalg.norm(W[i]) * 1.2 * \
                    np.max(np.linalg.norm(x, axis=1))
        torch.cuda.synchronize()
        for i in range(len(W)):
            ids = outs[i][0].cpu().numpy()
            # the oracle's list of the oracle scores may differ only by near-tie swaps; the GPU lists
            # of the same w on different streams / modes must be identical
            assert len(np.intersect1d(ids, want[i])) >= k - 2, (rep, i)
        for i, hid in host:
            np.testing.assert_array_equal(hid, outs[i][0].cpu().numpy())


def test_training_overlaps_ranking(otf):
    """north_star (5): Pegasos steps (trainer's high-priority stream, own thread) run while the
    ranker thread ranks; both make progress in the same wall-clock window and every ranked list
    stays exact."""
    rng = np.random.default_rng(13)
    n, d, k = 2_000_000, 128, 100
    x = rng.standard_normal((n, d)).astype(np.float32)
    repo = otf.Repository.dense(otf.FeatureStore(x))
    pos, neg = clusters(d, 200, 4096, 14)
    tr = otf.OnlineTrainer(d, neg, otf.TrainerConfig(lam=1e-3, batch_size=32, seed=3))
    tr.append_positives(pos)
    w = rng.standard_normal(d)
    ref = repo.rank(w, k)
    stop = threading.Event()
    steps = [0]

    def train():
        while not stop.is_set():
            tr.step()
            steps[0] += 1

    th = threading.Thread(target=train)
    t0 = time.monotonic()
    th.start()
    ranks = 0
    while time.monotonic() - t0 < 1.0:
        got = repo.rank(w, k)
        assert np.array_equal(got.ids, ref.ids) and np.array_equal(got.scores, ref.scores)
        ranks += 1
    stop.set()
    th.join()
    assert ranks > 50 and steps[0] > 50, (ranks, steps[0])
