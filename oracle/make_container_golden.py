"""Generate tests/golden/container_tiny/ with the REFERENCE's own
``write_container`` (gfmkit/container.py:124-183).  Test infrastructure only.

    PYTHONPATH=/root/reference/pkg/src python oracle/make_container_golden.py

Records: oracle synthetic(8, seed=21) (the reference's generate_synthetic
rng sequence), tags "s0".."s7"; groups trainset 0-4, valset 5-6, testset 7;
two sub-files.
"""
from __future__ import annotations

import os
import shutil
import sys

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
OUT = os.path.join(ROOT, "tests", "golden", "container_tiny")


def main() -> None:
    sys.path.insert(0, "/root/reference/pkg/src")
    sys.path.insert(0, ROOT)
    from gfmkit.container import write_container
    from gfmkit.records import GraphRecord

    from oracle import gfm_oracle as O

    recs = [GraphRecord(d["z"], d["pos"], d["edges"].astype(np.uint32), d["energy"], d["forces"],
                        f"s{i}") for i, d in enumerate(O.synthetic(8, seed=21))]
    shutil.rmtree(OUT, ignore_errors=True)
    write_container({"trainset": recs[:5], "valset": recs[5:7], "testset": recs[7:]}, 2, OUT)
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
