"""The C++ drop-in TieredKvCache (include/scout_b200_tier.hpp: the tier state
machine on the B200) beside the reference's own scout::TieredKvCache, compiled
from /root/reference into one binary by tests/cpp/Makefile
(tests/cpp/test_tier_cache.cpp): the reference's kv_store scenarios and random
operation sequences, compared after every operation."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
EXE = ROOT / "tests" / "cpp" / "_bin" / "test_tier_cache"


def test_cpp_tiered_kv_cache_vs_reference(cuda):
    assert EXE.exists(), f"{EXE} missing: build it with __graft_entry__.build() where /root/reference exists"
    r = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0 and "ALL PASS" in r.stdout, r.stdout[-4000:] + r.stderr[-2000:]
