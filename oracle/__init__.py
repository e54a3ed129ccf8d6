"""CPU oracle for the semisort / collect-reduce / histogram hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2304_10078_b200`` imports this
package; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may use it, and only as the
checker (or the timed CPU baseline), never as the product path.

Parity pin: ``tests/golden/make_golden.py`` runs the unmodified reference
package (``/root/reference/pkg/src/semisort``) in this container and commits
its outputs as fixtures; ``tests/test_oracle_golden.py`` asserts that this
restatement reproduces every one of them byte for byte.
"""

from .semisort_oracle import *  # noqa: F401,F403
from .checkers import *  # noqa: F401,F403
from .graphs_oracle import csr_from_edges, transpose as graph_transpose  # noqa: F401
from .records_oracle import dump_bytes, pack_rows, parse_dump  # noqa: F401
from .bytes_oracle import hash_bytes, semisort_bytes  # noqa: F401
