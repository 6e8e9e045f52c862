"""C1 at full BASELINE size, run through the REAL reference (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_c1.py

BASELINE.json configs[0]: 1M x 128-D synthetic CNN-M-128 features, a linear SVM trained on 200
positives + 16k fixed negatives, the full set ranked, top-1000. The reference pipeline is

    generate_corpus_bundle(SynthConfig(dim=128, classes=5, per_class=200, distractors=999_000,
                                       seed=S), train_per_class=200, negative_count=16_000)
                                                                          (store.py:324-362)
    train_batch(train rows of class 0, negatives, BatchTrainConfig(c=0.25))  (trainer.py:204-257)
    Repository.dense(test).rank(model, 1000)                                (ranker.py:272-281)

Only the small outputs are committed (tests/golden/golden_c1.npz): CRC32 checksums of the three
generated stores (so the oracle's port of generate_corpus_bundle is pinned without shipping 512
MB), the trained w, and the top-1000 ids and scores. The GPU test regenerates the corpus with the
oracle port, checks the checksums, trains with the package's train_batch and ranks on the GPU.
"""

from __future__ import annotations

import sys
import time
import zlib
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "golden_c1.npz"

C1 = dict(dim=128, classes=5, per_class=200, distractors=999_000, train_per_class=200, negatives=16_000,
          c=0.25, k=1000)
SEEDS = (1407, 4764)


def crc(a: np.ndarray) -> int:
    return zlib.crc32(np.ascontiguousarray(a).tobytes())


def main() -> None:
    sys.path.insert(0, str(REF))
    sys.dont_write_bytecode = True
    from otf_retrieval import ranker as rr
    from otf_retrieval import trainer as rt
    from otf_retrieval.store import SynthConfig, generate_corpus_bundle

    g: dict[str, np.ndarray] = {}
    for seed in SEEDS:
        t0 = time.perf_counter()
        cfg = SynthConfig(dim=C1["dim"], classes=C1["classes"], per_class=C1["per_class"],
                          distractors=C1["distractors"], seed=seed)
        b = generate_corpus_bundle(cfg, C1["train_per_class"], C1["negatives"])
        pos_rows = sorted(b.train_labels.ids_for("class_00"))
        pos = b.train.data[pos_rows]
        t1 = time.perf_counter()
        model = rt.train_batch(pos, b.negatives.data, rt.BatchTrainConfig(c=C1["c"]))
        t2 = time.perf_counter()
        repo = rr.Repository.dense(b.test)
        ranked = repo.rank(model, C1["k"])
        t3 = time.perf_counter()
        s = f"s{seed}"
        g[f"{s}_crc_test"] = np.array([crc(b.test.data)], dtype=np.int64)
        g[f"{s}_crc_train"] = np.array([crc(b.train.data)], dtype=np.int64)
        g[f"{s}_crc_neg"] = np.array([crc(b.negatives.data)], dtype=np.int64)
        g[f"{s}_crc_ids"] = np.array([crc(b.test.ids)], dtype=np.int64)
        g[f"{s}_pos_rows"] = np.asarray(pos_rows, dtype=np.int64)
        g[f"{s}_w"] = model.weights
        g[f"{s}_iter"] = np.array([model.iteration], dtype=np.int64)
        g[f"{s}_rank_ids"] = ranked.ids
        g[f"{s}_rank_scores"] = ranked.scores
        # the reference's own scores of the returned rows: the GPU test's tolerance baseline
        g[f"{s}_rank_names"] = np.array(ranked.names[:20])
        print(f"seed {seed}: corpus {t1 - t0:.1f}s train {t2 - t1:.1f}s rank {t3 - t2:.2f}s "
              f"top ids {ranked.ids[:5]} relevant in top-1000: {int(np.sum(ranked.ids < 1000))}")
    np.savez_compressed(OUT, **g)
    print("wrote", OUT, OUT.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
