"""Golden byte strings of the reference's inter-rank codecs (kdknn.wire) for fixed
inputs; run here with the reference importable:
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_wire_golden.py
Writes tests/golden/wire.npz (byte arrays) used by tests/test_dataset.py."""
import os

import numpy as np
from kdknn import wire
from kdknn.core import PointSet

rng = np.random.default_rng(77)
coords = rng.random((3, 11))
ids = rng.integers(0, 2**63, 11, dtype=np.uint64)
ps = PointSet(coords, ids)
q = rng.random((5, 3))
qid = np.arange(100, 105, dtype=np.uint64)
rp = rng.random(5)
cnt = np.array([2, 0, 3, 1, 2])
dd = rng.random(8)
pp = rng.integers(0, 2**40, 8, dtype=np.uint64)
rk = rng.integers(0, 8, 8)
out = {
    "points": wire.encode_points(ps), "queries": wire.encode_queries(qid, q),
    "requests": wire.encode_requests(qid, rp, q, 7), "responses": wire.encode_responses(qid, cnt, dd, pp, rk),
}
out["frame"] = wire.pack_frame(wire.KIND_REQUESTS, 6, out["requests"])
here = os.path.dirname(os.path.abspath(__file__))
np.savez(os.path.join(here, "wire.npz"), coords=coords, ids=ids, q=q, qid=qid, rp=rp, cnt=cnt, dd=dd, pp=pp, rk=rk,
         **{f"bytes_{k}": np.frombuffer(v, dtype=np.uint8) for k, v in out.items()})
print({k: len(v) for k, v in out.items()})
