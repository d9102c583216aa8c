"""Threads sharing one fresh matrix: every result must equal the reference's."""
import sys; sys.path.insert(0, '/root/repo')
import numpy as np
from concurrent.futures import ThreadPoolExecutor
import paper_2201_08560_b200 as b2
g = dict(np.load('/root/repo/tests/golden/golden.npz'))  # loaded up front: the npz reader is not thread-safe
name = "rmat10"
csr = b2.CsrMatrix(len(g[f"{name}/row_ptr"]) - 1, g[f"{name}/row_ptr"], g[f"{name}/col_ind"])
for d in (4, 8):
    for kind in ("bbb", "bff", "bbf", "mix"):
        bad = 0
        for rep in range(5):
            m = b2.csr_to_b2sr(csr, d)
            xb = b2.BitVector.from_bools(g[f"{name}/xb"], d)
            f_bbb = lambda: np.array_equal(b2.bmv_bin_bin_bin(m, xb).words, g[f"{name}/d{d}/bbb"])
            f_bff = lambda: b2.bmv_bin_full_full(m, g[f"{name}/xf"], b2.ARITHMETIC).tobytes() == g[f"{name}/d{d}/bff_ar"].tobytes()
            f_bbf = lambda: b2.bmv_bin_bin_full(m, xb).tobytes() == g[f"{name}/d{d}/bbf"].tobytes()
            jobs = {"bbb": [f_bbb] * 12, "bff": [f_bff] * 12, "bbf": [f_bbf] * 12, "mix": [f_bbb, f_bff, f_bbf] * 4}[kind]
            with ThreadPoolExecutor(max_workers=6) as ex:
                res = list(ex.map(lambda f: f(), jobs))
            bad += res.count(False)
        print(d, kind, "bad", bad, flush=True)
