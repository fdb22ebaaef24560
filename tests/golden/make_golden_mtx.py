"""Matrix Market fixtures + the REFERENCE reader's results on them (harness.py:138-220).
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_mtx.py
Writes tests/golden/mtx/*.mtx and tests/golden/golden_mtx.npz (committed)."""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
from densolve.harness import MatrixMarketError, read_matrix_market  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
D = os.path.join(HERE, "mtx")

rng = np.random.default_rng(2024)
S = rng.uniform(-1, 1, (5, 5))
S = S + S.T
FILES = {
    "array_1x1": "%%MatrixMarket matrix array real general\n1 1\n5.0\n",
    "array_colmajor": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "array_rect": "%%MatrixMarket matrix array real general\n% a comment\n\n3 2\n1.5\n-2e-3\n3\n+4\n5E1\n-0.0\n",
    "array_symmetric": "%%MatrixMarket matrix array real symmetric\n3 3\n1\n2\n3\n4\n5\n6\n",
    "array_sym_rand": "%%MatrixMarket matrix array real symmetric\n5 5\n" + "".join(
        f"{float(S[i, j])!r}\n" for j in range(5) for i in range(j, 5)),
    "coord_diag": "%%MatrixMarket matrix coordinate real general\n3 3 3\n1 1 1.0\n2 2 2.0\n3 3 3.0\n",
    "coord_sym": "%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n2 1 7.0\n",
    "coord_dup_last_wins": "%%MatrixMarket matrix COORDINATE REAL GENERAL\n2 2 3\n1 1 1\n1 1 2\n2 2 inf\n",
    "coord_comments": "%%MatrixMarket matrix coordinate real general\n%c1\n   \n2 3 2\n% mid\n1 3 -1.25\n2 1 1e300\n",
    # errors
    "err_empty": "",
    "err_header": "%%NotMatrixMarket\n1 1\n5.0\n",
    "err_complex": "%%MatrixMarket matrix array complex general\n1 1\n5 0\n",
    "err_pattern": "%%MatrixMarket matrix coordinate pattern general\n1 1 1\n1 1\n",
    "err_hermitian": "%%MatrixMarket matrix array real hermitian\n1 1\n5\n",
    "err_format": "%%MatrixMarket matrix dense real general\n1 1\n5\n",
    "err_no_size": "%%MatrixMarket matrix array real general\n% only comments\n\n",
    "err_bad_size": "%%MatrixMarket matrix array real general\n2 x\n1\n",
    "err_bad_size_coord": "%%MatrixMarket matrix coordinate real general\n2 2\n1 1 1\n",
    "err_count_array": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n",
    "err_count_coord": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n",
    "err_range": "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
    "err_value_coord": "%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 abc\n",
    "err_value_array": "%%MatrixMarket matrix array real general\n1 2\n1.0\nxyz\n",
    "err_entry_shape": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n",
    "err_float_index": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1.0 1 1\n",
    "err_hex": "%%MatrixMarket matrix array real general\n1 1\n0x1p3\n",
}


def main():
    os.makedirs(D, exist_ok=True)
    g = {}
    for name, text in FILES.items():
        path = os.path.join(D, name + ".mtx")
        with open(path, "w") as fh:
            fh.write(text)
        try:
            A = read_matrix_market(path)
            g[f"{name}_A"] = A
        except MatrixMarketError as e:
            g[f"{name}_err_line"] = np.asarray(e.line)
            g[f"{name}_err_msg"] = np.asarray(str(e))
    g["names"] = np.asarray(sorted(FILES))
    np.savez_compressed(os.path.join(HERE, "golden_mtx.npz"), **g)
    print("wrote", len(FILES), "fixtures")


if __name__ == "__main__":
    main()
