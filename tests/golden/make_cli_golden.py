"""Golden CSVs from the REFERENCE CLI (``particula md``, ref cli.py:173-206).

Run in the build container (where /root/reference exists):

    python tests/golden/make_cli_golden.py

Each case runs the unchanged reference CLI in a subprocess
(``PYTHONPATH=/root/reference/pkg/src python -m particula.cli md ...``) and
freezes its CSV as ``tests/golden/cli_<case>.csv``; tests/test_cli.py runs
the drop-in CLI with the same arguments and compares the ``#`` echo line and
the header byte for byte and the values within tolerance.  The phase-timing
sidecar is not frozen (timings are machine-bound).
"""

from __future__ import annotations

import os
import subprocess
import sys
import tempfile

OUT = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"

CASES = {
    # fcc 4^3 (256 atoms), skin + deferred rebuild
    "md_4": ["--lattice-cells", "4", "--steps", "20", "--temperature", "1.44", "--skin", "0.3",
             "--rebuild-stride", "5"],
    # fcc 6^3 (864 atoms) on the reference's simulated 2x2x1 fabric, locality sort
    "md_6_ranks": ["--lattice-cells", "6", "--steps", "10", "--temperature", "1.44",
                   "--skin", "0.3", "--rebuild-stride", "5", "--sort-stride", "5",
                   "--ranks", "2,2,1", "--seed", "7"],
}


def main():
    env = dict(os.environ, PYTHONPATH=REF_SRC, PYTHONDONTWRITEBYTECODE="1")
    with tempfile.TemporaryDirectory() as tmp:
        for name, args in CASES.items():
            path = os.path.join(tmp, f"{name}.csv")
            subprocess.run([sys.executable, "-m", "particula.cli", "md", *args, "--output", path],
                           check=True, env=env, cwd=tmp)
            with open(path, "rb") as fh:
                data = fh.read()
            with open(os.path.join(OUT, f"cli_{name}.csv"), "wb") as fh:
                fh.write(data)
            print(name, len(data.splitlines()), "lines")


if __name__ == "__main__":
    main()
