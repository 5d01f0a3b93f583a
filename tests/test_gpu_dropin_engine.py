"""The drop-in proof on the B200: the reference's own ScoutEngine with only the
INTEGRATION.md §1 call swaps (select_topk, partial_attention, merge, finalize
-> scout_b200::, generated from the unmodified engine.hpp by tests/cpp/Makefile)
against the unmodified reference engine and its oracles, linked in one binary
(tests/cpp/test_dropin_engine.cpp). Built in the build container by
__graft_entry__.build() (it compiles the reference headers); the binary
travels with the repo."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
EXE = ROOT / "tests" / "cpp" / "_bin" / "test_dropin_engine"


def test_reference_engine_with_scout_b200_call_swaps(cuda):
    assert EXE.exists(), f"{EXE} missing: build it with __graft_entry__.build() where /root/reference exists"
    r = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0 and "ALL PASS" in r.stdout, r.stdout[-4000:] + r.stderr[-2000:]
