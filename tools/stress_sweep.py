"""Long randomised sweep (760 cases) over the rank / rank_many / pq_encode paths through the C ABI,
reusing the case generators of tests/test_gpu_random_sweep.py. Run on a GPU box:
    python tools/stress_sweep.py
"""
import sys
sys.path.insert(0, "tests"); sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
import numpy as np
import paper_1407_4764_b200 as otf
import test_gpu_random_sweep as T
bad = 0
for seed in range(1000, 1600):
    try:
        T.test_random_rank(otf, seed)
    except AssertionError as e:
        bad += 1
        print("FAIL rank", seed, str(e)[:200])
for seed in range(3000, 3060):
    try:
        T.test_random_rank_many(otf, seed)
    except AssertionError as e:
        bad += 1
        print("FAIL many", seed, str(e)[:200])
for seed in range(5000, 5100):
    try:
        T.test_random_pq_encode(otf, seed)
    except AssertionError as e:
        bad += 1
        print("FAIL enc", seed, str(e)[:200])
print("stress done, failures:", bad)
