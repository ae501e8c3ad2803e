"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference sources (compiled into oracle/_ref/ by
oracle/Makefile) — never our code — and stores inputs plus outputs:
  * workload_*.npz : generate_workload outputs (workload.cpp:102-203)
  * graph_*.oodg   : OODG v1 blobs from ood_build (index_oodgraph.cpp:89-355)
  * search_*.npz   : OODGraph::search results (ids, scores, scanned, truncated)
                     for decode queries x {no mask, static W} x ef grid
  * attn_*.npz     : partial_attention over W and Omega + merge per query
Re-run: python tests/golden/make_golden.py   (needs /root/reference)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.ffi import BuildParams, Oracle  # noqa: E402

CASES = {
    # name: (n_ctx, d_model, d_head, n_heads, n_groups, seed, n_decode, params)
    "d32": (2048, 64, 32, 2, 1, 7, 8, BuildParams(k_train=32, max_degree=16, ef_construction=64)),
    "d128": (2048, 256, 128, 1, 1, 8, 8,
             BuildParams(k_train=128, max_degree=24, ef_construction=256, edge_window=8)),
}
EFS = [16, 64, 128]


def main():
    R = Oracle("ref")
    for name, (n, dm, dh, H, G, seed, nd, bp) in CASES.items():
        w = R.generate_workload(n, dm, dh, H, G, seed=seed, n_decode=nd)
        np.savez_compressed(os.path.join(HERE, f"workload_{name}.npz"),
                            spec=np.array([n, dm, dh, H, G, seed, nd], np.int64), **w)
        W, _ = R.static_partition(n, 128, 512)
        for h in range(H):
            g = h // (H // G)
            blob = R.graph_build(w["keys"][g], w["prefill_q"][h], bp)
            with open(os.path.join(HERE, f"graph_{name}_h{h}.oodg"), "wb") as f:
                f.write(blob)
            G_ = R.graph(w["keys"][g], blob)
            rows = []
            for qi in range(nd):
                q = w["decode_q"][h][qi]
                for mi, mask in enumerate([None, W]):
                    for ef in EFS:
                        k = min(100, ef)
                        r = G_.search(q, k, mask, ef)
                        ids = np.full(100, 0xFFFFFFFF, np.uint32)
                        sc = np.full(100, np.nan, np.float32)
                        ids[: len(r.ids)] = r.ids
                        sc[: len(r.scores)] = r.scores
                        rows.append((qi, mi, ef, k, ids, sc, r.scanned, r.truncated))
            np.savez_compressed(
                os.path.join(HERE, f"search_{name}_h{h}.npz"),
                qi=np.array([r[0] for r in rows]), mask=np.array([r[1] for r in rows]),
                ef=np.array([r[2] for r in rows]), k=np.array([r[3] for r in rows]),
                ids=np.stack([r[4] for r in rows]), scores=np.stack([r[5] for r in rows]),
                scanned=np.array([r[6] for r in rows]),
                truncated=np.array([r[7] for r in rows]))
            # engine run_head pieces at top_k 100, default ef 128
            outs, zw, sw, zo, so, om = [], [], [], [], [], []
            for qi in range(nd):
                q = w["decode_q"][h][qi]
                r = G_.search(q, 100, W, 128)
                pw = R.partial_attention(q, w["keys"][g], w["values"][g], W)
                po = R.partial_attention(q, w["keys"][g], w["values"][g], r.ids)
                out, _, _ = R.merge(pw, po, dh)
                outs.append(out)
                zw.append(pw[1]); sw.append(pw[2]); zo.append(po[1]); so.append(po[2])
                o = np.full(100, 0xFFFFFFFF, np.uint32)
                o[: len(r.ids)] = r.ids
                om.append(o)
            np.savez_compressed(os.path.join(HERE, f"attn_{name}_h{h}.npz"),
                                out=np.stack(outs), zw=np.array(zw), sw=np.array(sw),
                                zo=np.array(zo), so=np.array(so), omega=np.stack(om))
        print("wrote", name)
    with open(os.path.join(HERE, "splitmix64.txt"), "w") as f:
        # util test golden (test_util.cpp:13-19) reproduced through the reference
        f.write(" ".join(str(x) for x in R.splitmix64(1234567, 3)) + "\n")


if __name__ == "__main__":
    main()
