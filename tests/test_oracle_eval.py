"""Oracle evaluation (oracle/oracle_eval.cpp) pinned by the reference's own
evaluation KATs (proj/tests/test_eval.cpp, acceptance.cpp:594-620)."""
import pytest

from oracle import oracle as O
from tests import eval_kats


@pytest.mark.parametrize("kat", eval_kats.ALL, ids=lambda f: f.__name__)
def test_oracle_eval_kat(kat):
    kat(O)
