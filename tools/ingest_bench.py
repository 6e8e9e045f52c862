"""§8(f3) loader throughput: a 100M x 16 OTFC file (1.6 GB) loaded into a PQ Repository
(Repository.load_quantized: chunked multi-threaded pread -> pinned staging -> H2D, then the code
range check on the device) against the host read bandwidth of the same reads with no device copy
(otf_file_read_bench), and against the reference's path (numpy load_pq_codes-equivalent read +
Repository.quantized from the host array).

    python tools/ingest_bench.py [rows] [dir]
"""
import ctypes as C
import os
import struct
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import paper_1407_4764_b200 as otf  # noqa: E402
from paper_1407_4764_b200 import _lib  # noqa: E402


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
    d = Path(sys.argv[2]) if len(sys.argv) > 2 else Path("/tmp")
    path = d / "ingest_bench.otfc"
    rng = np.random.default_rng(0)
    cents = rng.standard_normal((16, 256, 8)).astype(np.float32)
    with open(path, "wb") as fh:
        fh.write(b"OTFC" + struct.pack("<I", 1) + struct.pack("<Q", rows) + struct.pack("<I", 16))
        step = 10_000_000
        for r0 in range(0, rows, step):
            fh.write(rng.integers(0, 256, (min(step, rows - r0), 16), dtype=np.uint8).tobytes())
    size = path.stat().st_size
    book = otf.PQCodebook(cents)
    lib = _lib.load()
    sec, nb = C.c_double(), C.c_int64()
    reads, loads, refs = [], [], []
    for _ in range(3):
        _lib.check(lib.otf_file_read_bench(str(path).encode(), 20, C.byref(sec), C.byref(nb)))
        reads.append(sec.value)
        t0 = time.perf_counter()
        repo = otf.Repository.load_quantized(book, path)
        loads.append(time.perf_counter() - t0)
        assert repo.count == rows
        del repo
    for _ in range(2):  # the reference's path: the whole payload into a host array, then the copy
        t0 = time.perf_counter()
        with open(path, "rb") as fh:
            fh.seek(20)
            codes = np.frombuffer(fh.read(), dtype=np.uint8).reshape(rows, 16).copy()
        repo = otf.Repository.quantized(book, codes)
        refs.append(time.perf_counter() - t0)
        del repo, codes
    gb = (size - 20) / 1e9
    r, l, f = min(reads), min(loads), min(refs)
    print(f"rows {rows} payload {gb:.2f} GB threads {os.environ.get('OTF_INGEST_THREADS', 4)}")
    print(f"host read (no device copy)  {r * 1e3:8.1f} ms  {gb / r:6.2f} GB/s")
    print(f"load_quantized (to HBM)     {l * 1e3:8.1f} ms  {gb / l:6.2f} GB/s  = {r / l:.2f} of the host read bandwidth")
    print(f"host array + quantized      {f * 1e3:8.1f} ms  {gb / f:6.2f} GB/s")
    path.unlink()


if __name__ == "__main__":
    main()
