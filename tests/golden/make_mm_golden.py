"""Golden vectors for the Matrix Market reader (io.py:114-199): every case
below is parsed by the REFERENCE reader (run in a container where
/root/reference exists) and its EdgeList -- or its ParseError message and
line -- stored in mm_cases.json.  tests/test_matrix_market.py replays them
through this package's reader.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_mm_golden.py
"""
import json
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import graphalg  # noqa: E402
from graphalg.errors import ParseError  # noqa: E402

HDR = "%%MatrixMarket matrix coordinate"
CASES = {
    "pattern_general": f"{HDR} pattern general\n% c\n4 4 3\n1 2\n2 3\n4 1\n",
    "pattern_symmetric": f"{HDR} pattern symmetric\n3 3 3\n1 2\n2 2\n3 1\n",
    "real_general": f"{HDR} real general\n3 3 2\n1 3 2.5\n3 2 -1e-3\n",
    "integer_symmetric": f"{HDR} integer symmetric\n%\n\n3 3 2\n2 1 7\n3 3 4\n",
    "rectangular": f"{HDR} real general\n2 5 2\n1 5 1.0\n2 4 0.5\n",
    "upper_case_field": f"{HDR} Pattern General\n2 2 1\n1 2\n",
    "blank_and_comment_lines": f"{HDR} pattern general\n%a\n\n2 2 2\n\n1 1\n% mid\n2 1\n",
    "extra_tokens": f"{HDR} pattern general\n2 2 1\n1 2 9 9\n",
    "empty_matrix": f"{HDR} pattern general\n5 5 0\n",
    # errors
    "err_empty": "",
    "err_banner": "%%MatrixMarket tensor coordinate pattern general\n1 1 0\n",
    "err_layout": "%%MatrixMarket matrix array real general\n1 1 1\n1\n",
    "err_field": f"{HDR} complex general\n1 1 0\n",
    "err_symmetry": f"{HDR} real hermitian\n1 1 0\n",
    "err_no_size": f"{HDR} real general\n% only comments\n",
    "err_size": f"{HDR} real general\n3 x 2\n",
    "err_fields": f"{HDR} real general\n3 3 1\n1 2\n",
    "err_entry": f"{HDR} real general\n3 3 1\n1 b 2.0\n",
    "err_range": f"{HDR} pattern general\n3 3 1\n4 1\n",
    "err_zero_index": f"{HDR} pattern general\n3 3 1\n0 1\n",
    "err_count": f"{HDR} pattern general\n3 3 3\n1 2\n2 3\n",
}


def main():
    out = {}
    with tempfile.TemporaryDirectory() as d:
        for name, text in CASES.items():
            p = os.path.join(d, name + ".mtx")
            with open(p, "w", encoding="ascii") as fh:
                fh.write(text)
            try:
                e = graphalg.read_matrix_market(p)
                out[name] = {"text": text, "n": int(e.n), "src": e.src.tolist(),
                             "dst": e.dst.tolist(),
                             "weight": None if e.weight is None else e.weight.tolist()}
            except ParseError as exc:
                out[name] = {"text": text, "error": str(exc), "line": exc.line}
    dst = os.path.join(os.path.dirname(os.path.abspath(__file__)), "mm_cases.json")
    with open(dst, "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print(f"wrote {len(out)} cases to {dst}")


if __name__ == "__main__":
    main()
