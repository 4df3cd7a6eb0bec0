"""Generate problem / solution file fixtures with the REFERENCE's own writer
(conesplit 0.1.0, fileio.py:170-187).  Build container only:

    python tests/golden/make_io_golden.py

Outputs (committed): io_problem.json (a small LP+SOC+PSD problem written by
conesplit.fileio.write_problem) and io_solution.json (its indirect solve,
written by conesplit.fileio.write_solution).
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from conesplit import fileio, generators  # noqa: E402
import conesplit as ref  # noqa: E402

data = generators.gen_rpca(3, 1, seed=2)
fileio.write_problem(os.path.join(HERE, "io_problem.json"), data)
sol = ref.solve(data, ref.Settings(linsys_mode="indirect"))
sol.info.solve_time = 0.0125  # fixed, so the fixture is reproducible
fileio.write_solution(os.path.join(HERE, "io_solution.json"), sol)
print(data.m, data.n, data.spec, sol.status)
