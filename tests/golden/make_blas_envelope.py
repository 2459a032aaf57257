"""How sensitive is the REFERENCE's own iteration count to summation order?

Run in the build container only (needs /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_blas_envelope.py

The long cfg1-geometry coupled solves (reference semantics, ~270 outer
iterations over ~9 restart cycles; golden ``solve_cfg1``) are chaotic in the
last bits of the dot products.  This script runs the *unmodified* reference
``harness.solve_coupled`` (harness.py:342-398) once per OpenBLAS CPU kernel
(``OPENBLAS_CORETYPE``: the same numpy / OpenBLAS 0.3.30 build, only the
SIMD ddot/dgemv kernel and therefore the reduction order differs -- what a
different host CPU would select) and records iterations / converged / final
residual.  ``tests/test_gpu_solve.py`` gates the device solve against this
envelope (the reference's own spread, +-2) instead of one host's count.
Writes ``blas_envelope_cfg1.npz``.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
CORETYPES = ("Prescott", "Nehalem", "Sandybridge", "Haswell", "SkylakeX", "Zen")

CHILD = r"""
import json, sys, tempfile
from pathlib import Path
sys.path.insert(0, {here!r})
import make_golden as MG
from mdprec import assembly, geometry, harness, neural
import numpy as np
assembly.refine_graph = MG.fixed_refine(32)
grid = geometry.StructuredGrid(17)
g = geometry.Graph1D(np.array([[0.5, 0.5, 0.1], [0.5, 0.5, 0.9]]), np.array([[0, 1]]), 0.02, (0,))
s = assembly.assemble_coupled_system(grid, g, MG.BetaParams(epsilon=0.02, beta=1.0), n_circle=8)
out = {{}}
with tempfile.TemporaryDirectory() as td:
    ck = Path(td) / "noisy0.mdu3"
    neural.save_checkpoint(MG.noisy_params(0), ck)
    for label, spec in (("none", {{"type": "none"}}),
                        ("neural_s", {{"type": "neural", "checkpoint": str(ck), "smoothing": {{"maxit": 2}}}})):
        st = harness.CoupledStrategy(tol=1e-6, maxit=300, restart=30, inner_iterations=3, one_d="ilu0",
                                     three_d=spec)
        _, _, rep = harness.solve_coupled(s, st)
        out[label] = [rep.iterations, bool(rep.converged), float(rep.rel_residual)]
print("RESULT " + json.dumps(out))
"""


def main():
    rows = {}
    for ct in CORETYPES:
        env = dict(os.environ, OPENBLAS_CORETYPE=ct, NUMBA_CACHE_DIR=os.environ.get("NUMBA_CACHE_DIR",
                                                                                     "/tmp/numba_cache"))
        p = subprocess.run([sys.executable, "-c", CHILD.format(here=str(HERE))], env=env, capture_output=True,
                           text=True, check=True)
        line = [ln for ln in p.stdout.splitlines() if ln.startswith("RESULT ")][-1]
        rows[ct] = json.loads(line[7:])
        print(ct, rows[ct], flush=True)
    out = {"coretypes": np.array(CORETYPES)}
    for label in ("none", "neural_s"):
        out[f"{label}_iters"] = np.array([rows[c][label][0] for c in CORETYPES])
        out[f"{label}_conv"] = np.array([rows[c][label][1] for c in CORETYPES])
        out[f"{label}_rel"] = np.array([rows[c][label][2] for c in CORETYPES])
    np.savez_compressed(HERE / "blas_envelope_cfg1.npz", **out)


if __name__ == "__main__":
    main()
