"""Debug aid: first mismatch of GPU search vs oracle on random graphs."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_10516_b200 as ra
from oracle.ffi import Oracle, BuildParams
port = Oracle("port")
rng = np.random.default_rng(11)
for n, d, M, nq in [(500, 16, 8, 100), (3000, 32, 16, 600), (1500, 128, 24, 300),
                    (700, 20, 12, 100), (64, 8, 32, 4)]:
    keys = rng.standard_normal((n, d)).astype(np.float32)
    tq = rng.standard_normal((nq, d)).astype(np.float32)
    blob = port.graph_build(keys, tq, BuildParams(k_train=min(32, n), max_degree=M, ef_construction=2 * M))
    g = ra.OODGraph.from_blob(ra.KVGroup(keys), blob)
    og = port.graph(keys, blob)
    Q = rng.standard_normal((40, d)).astype(np.float32)
    mask = np.sort(rng.choice(n, size=n // 5, replace=False)).astype(np.uint32)
    bad = 0
    for mi, m in enumerate((None, mask)):
        for ef, k in ((10, 10), (64, 20), (200, 100), (n, min(n, 300))):
            res = ra.search_batch([g], Q, k, m, ef).host()
            for qi in range(len(Q)):
                a, b = res[qi], og.search(Q[qi], k, m, ef)
                if not (np.array_equal(a.ids, b.ids) and a.scanned == b.scanned and a.truncated == b.truncated):
                    bad += 1
                    if bad <= 3:
                        print(f"n={n} d={d} M={M} mask={mi} ef={ef} k={k} q={qi}: scanned {a.scanned} vs {b.scanned}, "
                              f"len {len(a.ids)} vs {len(b.ids)}, first diff at "
                              f"{next((i for i in range(min(len(a.ids), len(b.ids))) if a.ids[i] != b.ids[i]), None)}")
    print(f"n={n} d={d} M={M}: mismatches {bad}")
