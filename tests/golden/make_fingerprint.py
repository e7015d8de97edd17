#!/usr/bin/env python3
"""The reference's backend-parity digest (pkg/tests/helpers.py:190-223,
`backend_fingerprint`, used by test_backends.py:36-41 to compare its numba
and interpreted backends) computed by the REFERENCE itself, numba backend.

Run in the build container (needs /root/reference):

    python tests/golden/make_fingerprint.py

Writes tests/golden/fingerprint.json; tests/test_gpu_parity.py::
test_reference_backend_fingerprint recomputes the same digest through this
package's API on the GPU and requires equality -- the CUDA backend dropped
into the reference's own backend-parity harness.
"""

import json
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REF / "src"), str(REF / "tests")]

from helpers import backend_fingerprint  # noqa: E402
from rcpsp_tabu import kernels  # noqa: E402

assert kernels.BACKEND == "numba", kernels.BACKEND
out = Path(__file__).resolve().parent / "fingerprint.json"
out.write_text(json.dumps(backend_fingerprint(), indent=0) + "\n")
print("wrote", out)
