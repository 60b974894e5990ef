"""CPU oracle for the H1 peeling hot path -- TEST INFRASTRUCTURE ONLY.

A plain numpy/scipy restatement of the reference library ``hpeel``
(arxiv 2205.03406) for the H1 path: RNG, box tree, adjacency, constraint
graph + DSatur, test-matrix realization, run_h1 / extract_leaf / compress,
H1Rep apply and the power-method error estimator. Every function cites the
reference file:line it follows (paths relative to /root/reference/).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU baseline
leg may import this package, and only as the checker / CPU reference arm.
The product path (``paper_2205_03406_b200``) never calls into it.

Pinning: the reference cannot be compiled here (Eigen3 and vendor/ are absent,
SURVEY.md 8(c)), so this restatement is pinned by the reference's own
known-answer and tolerance tests (proj/tests/test_box_tree.cpp,
test_coloring.cpp, test_peeling.cpp, test_linalg.cpp) restated in
tests/test_oracle.py, and by the frozen RNG algorithm text
(proj/include/hpeel/rng.hpp:12-17, :44-48). Eigen's ColPivHouseholderQR and
BDCSVD are replaced by LAPACK dgeqp3 (scipy) and dgesdd (numpy): same
algorithms up to near-tie pivots and singular-vector signs, so individual
factor values are not pinned; spans, U B V^T and errors are.
"""
from .hpeel_ref import *  # noqa: F401,F403
