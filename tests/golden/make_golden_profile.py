"""Golden reports of the REFERENCE tile-width sampler (b2sr.sample_profile,
profile.py:73-127), for the GPU sampler's parity test.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_profile.py

Inputs: every case of golden.npz, plus R-MAT scale 12 and 14 graphs from the
oracle's CPU generator; sample counts 1, 7, 100 and ceil(n/4) (clipped to
the valid range), seeds 0 and 5.  Output: golden_profile.json.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))

import b2sr  # noqa: E402  (the reference, not this repo)

assert "reference" in b2sr.__file__, b2sr.__file__

from oracle import oracle  # noqa: E402


def main():
    g = np.load(HERE / "golden.npz")
    names = [c["name"] for c in json.load(open(HERE / "manifest.json"))["cases"]]
    graphs = {nm: (g[f"{nm}/row_ptr"], g[f"{nm}/col_ind"]) for nm in names}
    for scale in (12, 14):
        graphs[f"rmat{scale}"] = oracle.rmat_csr(scale, 16, seed=1)
    out = []
    for nm, (rp, ci) in graphs.items():
        n = len(rp) - 1
        csr = b2sr.CsrMatrix(n, rp, ci)
        max_rows = (n + 3) // 4
        for count in sorted({1, 7, 100, max_rows}):
            if not 1 <= count <= max_rows:
                continue
            for seed in (0, 5):
                rep = b2sr.sample_profile(csr, count, seed).to_report()
                out.append({"graph": nm, "sample_count": count, "seed": seed, "report": rep})
    (HERE / "golden_profile.json").write_text(json.dumps(out, indent=0, sort_keys=False))
    print(len(out), "reports")


if __name__ == "__main__":
    main()
