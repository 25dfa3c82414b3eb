"""Golden for cases.cfg3_default() made by running the REFERENCE itself
(nervemap.compute_mapper with its default strategy, 8 fork workers) in the
build container. ~1 h on 8 cores: 5 elements of 20-22k rows take the
on-the-fly path (2 numpy distance rows per point).

    python tests/golden/make_golden_cfg3d.py
"""

from __future__ import annotations

import os
import sys
import time

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as mg  # noqa: E402  (puts /root/reference/pkg/src on the path)
import cases  # noqa: E402


def main():
    t = time.time()
    X, p = cases.cfg3_default()
    g = mg.run(X, p, threads=os.cpu_count() or 1)
    mg.save("cfg3d", x_sha=mg.np.array(cases.sha(X)), **mg.compact("graph", g))
    print("cfg3d", time.time() - t, flush=True)


if __name__ == "__main__":
    main()
