"""Live query sessions on one GPU — the caller of the hot path (reference session.py:44-290).

The reference session (feed positives, train continuously, re-rank every tau) is reused
semantically, with the state where the GPU needs it:
  * the positive pool lives in the trainer's HBM pool (``PositivePool``, session.py:62-93), so a
    training step gathers its B/2 positives on the device instead of converting the whole pool to
    float64 on the host every step (trainer.py:100-102);
  * ``train_step`` runs one Pegasos kernel on the trainer's high-priority stream;
  * ``rank_tick`` publishes w into the trainer's own snapshot buffer on the device
    (``OnlineTrainer.publish_to``: one device copy ordered on the trainer stream + a CUDA event —
    no host round trip; versioned exactly like trainer.py:161-173), then ranks the GPU-resident
    repository under that snapshot (``Repository.rank_published(trainer, ...)``: the ranker's
    stream waits for the event; the snapshot is per trainer, so sessions sharing a repository
    never rank under each other's w); the publication carries the same CRC32 over the int64 ids /
    float64 scores bytes as session.py:96-116.
``run_simulated`` replays a session on a virtual clock with the reference's event order
(feeds at (i+1)/rate, training every 1/steps_per_second from the first arrival, rank ticks
every interval; feed < train < rank at equal times — session.py:237-290). ``WallRunner`` is the
wall-clock driver (session.py:295-359): feeder, trainer and ranker threads around one session.
"""

from __future__ import annotations

import dataclasses
import heapq
import threading
import time
import zlib

import numpy as np

from .errors import ConfigError, NotReadyError
from .ranker import RankedList, RankerConfig
from .trainer import OnlineTrainer, TrainerConfig

DEFAULT_FEED_RATE = 12.0
DEFAULT_STEPS_PER_SECOND = 500.0
STATE_WARMING, STATE_TRAINING, STATE_STOPPED, STATE_FAILED = "warming", "training", "stopped", "failed"
_FEED, _TRAIN, _RANK = 0, 1, 2


@dataclasses.dataclass(frozen=True)
class SessionConfig:
    """session.py:44-59."""

    rate: float = DEFAULT_FEED_RATE
    ranker: RankerConfig = dataclasses.field(default_factory=RankerConfig)
    trainer: TrainerConfig = dataclasses.field(default_factory=TrainerConfig)
    steps_per_second: float = DEFAULT_STEPS_PER_SECOND

    def validate(self) -> None:
        if self.rate < 0:
            raise ConfigError(f"rate must be >= 0, got {self.rate}")
        if self.steps_per_second <= 0:
            raise ConfigError(f"steps_per_second must be positive, got {self.steps_per_second}")
        self.ranker.validate()
        self.trainer.validate()


@dataclasses.dataclass(frozen=True)
class Publication:
    """session.py:96-116 — a published list plus counters, CRC32 over its exact bytes."""

    ranked: RankedList
    positives_fed: int
    steps_applied: int
    lists_published: int
    checksum: int

    @staticmethod
    def crc(ranked: RankedList) -> int:
        c = zlib.crc32(np.ascontiguousarray(ranked.ids, dtype=np.int64).tobytes())
        c = zlib.crc32(np.ascontiguousarray(ranked.scores, dtype=np.float64).tobytes(), c)
        return zlib.crc32(str(ranked.model_version).encode(), c)

    @classmethod
    def build(cls, ranked: RankedList, positives_fed: int, steps_applied: int, lists_published: int):
        return cls(ranked, positives_fed, steps_applied, lists_published, cls.crc(ranked))

    def verify_checksum(self) -> bool:
        return self.checksum == self.crc(self.ranked)


class PoolView:
    """What ``PositivePool.snapshot()`` hands the trainer: a row count over the device pool."""

    def __init__(self, pool: "PositivePool", count: int):
        self.pool, self.count = pool, count

    def __len__(self) -> int:
        return self.count


class PositivePool:
    """session.py:62-93 — append-only float32 positives, stored in the trainer's HBM pool."""

    def __init__(self, dim: int, trainer: OnlineTrainer):
        self._dim = int(dim)
        self._trainer = trainer
        self._count = 0
        self._lock = threading.Lock()

    def __len__(self) -> int:
        return self._count

    def append(self, vector) -> int:
        vec = np.asarray(vector, dtype=np.float32)
        if vec.shape != (self._dim,):
            raise ConfigError(f"vector shape {vec.shape} does not match pool dim {self._dim}")
        # the library call runs outside the pool lock: a feeder waiting for the GIL after the
        # call must not hold the lock the trainer's snapshot() needs
        n = self._trainer.append_positives(vec[np.newaxis, :])
        with self._lock:
            self._count = max(self._count, n)
            return self._count

    def snapshot(self) -> PoolView:
        with self._lock:
            return PoolView(self, self._count)


class QuerySession:
    """session.py:119-232 — one live query: device pool, GPU trainer, published list."""

    def __init__(self, session_id: str, query_text: str, repository, adapted_negatives, cfg: SessionConfig,
                 trainer_seed: int = 0, created_at: float = 0.0):
        cfg.validate()
        self.id, self.query_text, self.cfg = session_id, query_text, cfg
        self.repository = repository
        self.created_at = created_at
        self.stopped_at: float | None = None
        self.failure: str | None = None
        self.trainer = OnlineTrainer(repository.model_dim, adapted_negatives,
                                     dataclasses.replace(cfg.trainer, seed=trainer_seed))
        self.pool = PositivePool(repository.model_dim, self.trainer)
        self._state = STATE_WARMING
        self._lock = threading.Lock()
        self._publication: Publication | None = None
        self._lists_published = 0
        self.publication_history: list[Publication] = []

    @property
    def state(self) -> str:
        with self._lock:
            return self._state

    @property
    def is_live(self) -> bool:
        return self.state in (STATE_WARMING, STATE_TRAINING)

    def mark_failed(self, reason: str, now: float = 0.0) -> None:
        with self._lock:
            self._state, self.failure, self.stopped_at = STATE_FAILED, reason, now

    def mark_stopped(self, now: float = 0.0) -> None:
        with self._lock:
            if self._state not in (STATE_FAILED, STATE_STOPPED):
                self._state, self.stopped_at = STATE_STOPPED, now

    def feed_one(self, vector) -> None:
        """session.py:181-187: adapt the raw positive (binary repos binarize on the GPU)."""
        adapted = self.repository.adapt_training_vectors(np.asarray(vector, dtype=np.float32))
        self.pool.append(adapted)
        with self._lock:
            if self._state == STATE_WARMING:
                self._state = STATE_TRAINING

    def train_step(self) -> bool:
        """session.py:189-195: one mini-batch over the device pool; False while it is empty."""
        if len(self.pool.snapshot()) == 0:
            return False
        self.trainer.step()
        return True

    def rank_tick(self, now: float) -> bool:
        """session.py:197-218: rank under the latest snapshot and publish the top k."""
        try:
            # device-side snapshot: w goes from the trainer's buffer to the ranker's on the GPU
            # (copy + event), versioned exactly like trainer.snapshot()
            _, version = self.trainer.publish_to(self.repository)
        except NotReadyError:
            return False
        ranked = self.repository.rank_published(self.trainer, self.cfg.ranker.k, produced_at=now,
                                                model_version=version)
        with self._lock:
            self._lists_published += 1
            pub = Publication.build(ranked, len(self.pool), self.trainer.iteration, self._lists_published)
            self._publication = pub
            self.publication_history.append(pub)
        return True

    def latest_publication(self) -> Publication | None:
        with self._lock:
            return self._publication

    def stats(self) -> dict:
        with self._lock:
            return {"positives_fed": len(self.pool), "steps_applied": self.trainer.iteration,
                    "lists_published": self._lists_published}


def run_simulated(session: QuerySession, vectors, duration: float, on_publish=None) -> None:
    """session.py:237-290 — the deterministic virtual-clock replay (same event order)."""
    cfg = session.cfg
    if duration <= 0:
        raise ConfigError(f"duration must be positive, got {duration}")
    vecs = np.asarray(vectors, dtype=np.float32)
    queue: list[tuple[float, int, int]] = []
    order = 0

    def push(at: float, kind: int) -> None:
        nonlocal order
        heapq.heappush(queue, (at, kind, order))
        order += 1

    if cfg.rate > 0:
        for i in range(len(vecs)):
            if (i + 1) / cfg.rate > duration:
                break
            push((i + 1) / cfg.rate, _FEED)
    for j in range(1, int(duration / cfg.ranker.interval + 1e-9) + 1):
        push(j * cfg.ranker.interval, _RANK)
    gap = 1.0 / cfg.steps_per_second
    training, fed = False, 0
    while queue:
        at, kind, _ = heapq.heappop(queue)
        if kind == _FEED:
            session.feed_one(vecs[fed])
            fed += 1
            if not training:
                push(at, _TRAIN)
                training = True
        elif kind == _TRAIN:
            session.train_step()
            if at + gap <= duration:
                push(at + gap, _TRAIN)
        elif session.rank_tick(at) and on_publish is not None:
            on_publish(session.latest_publication())
    session.mark_stopped(duration)


class WallRunner:
    """session.py:295-359 — the wall-clock driver: a feeder, a trainer and a ranker thread around
    one session. Each role is a plain loop on the monotonic clock; ctypes releases the GIL inside
    every library call, so the trainer's Pegasos kernels (high-priority stream) and the ranker's
    scans overlap on the GPU. ``stop`` is idempotent and leaves the session stopped."""

    def __init__(self, session: QuerySession, vectors):
        self.session = session
        self._vectors = np.asarray(vectors, dtype=np.float32)
        self._halt = threading.Event()
        roles = (("feeder", self._feed), ("trainer", self._train), ("ranker", self._rank))
        self._threads = [threading.Thread(target=fn, name=f"{role}-{session.id}", daemon=True) for role, fn in roles]
        self.errors: list[BaseException] = []

    def start(self) -> None:
        for th in self._threads:
            th.start()

    def stop(self) -> None:
        self._halt.set()
        me = threading.current_thread()
        for th in self._threads:
            if th is not me and th.ident is not None:
                th.join(timeout=5.0)
        self.session.mark_stopped(time.monotonic())

    def _guard(self, body) -> None:
        try:
            body()
        except BaseException as exc:  # a failing role fails the session, as a crashed thread would
            self.errors.append(exc)
            self.session.mark_failed(repr(exc), time.monotonic())
            self._halt.set()

    def _feed(self) -> None:
        def body():
            rate = self.session.cfg.rate
            if rate <= 0:
                return
            t0 = time.monotonic()
            for i, vec in enumerate(self._vectors):
                wait = t0 + (i + 1) / rate - time.monotonic()
                if (wait > 0 and self._halt.wait(wait)) or self._halt.is_set():
                    return
                self.session.feed_one(vec)
        self._guard(body)

    def _train(self) -> None:
        def body():
            gap = 1.0 / self.session.cfg.steps_per_second
            while not self._halt.is_set():
                t = time.monotonic()
                if not self.session.train_step():
                    self._halt.wait(0.005)
                    continue
                rest = gap - (time.monotonic() - t)
                if rest > 0:
                    self._halt.wait(rest)
        self._guard(body)

    def _rank(self) -> None:
        def body():
            interval = self.session.cfg.ranker.interval
            due = time.monotonic() + interval
            while True:
                wait = due - time.monotonic()
                if (wait > 0 and self._halt.wait(wait)) or self._halt.is_set():
                    return
                self.session.rank_tick(time.monotonic())
                now = time.monotonic()
                due += interval
                if due < now:  # a slow tick skips the missed ticks instead of queueing them
                    due = now + interval
        self._guard(body)
