"""The C-ABI library loads on a CPU-only host and exports exactly what
include/treeserve_b200.h declares (no compute calls: no GPU here)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "treeserve_b200.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int64_t|int|const char\*)\s+(ts_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__ as g

    g.build()
    from paper_2604_00510_b200._abi import load_library

    return load_library()


def test_header_and_mirror_agree():
    from paper_2604_00510_b200._abi import EXPORTED

    assert sorted(EXPORTED) == _declared()


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.ts_abi_version() == 6


def test_struct_layouts_match_header():
    from paper_2604_00510_b200._abi import TsConfig, TsOutcome, TsProblem, TsSchedRecord
    from oracle import oracle

    L = oracle.lib()
    assert L.or_sizeof_problem() == ctypes.sizeof(TsProblem)
    assert L.or_sizeof_config() == ctypes.sizeof(TsConfig)
    assert L.or_sizeof_outcome() == ctypes.sizeof(TsOutcome)
    assert ctypes.sizeof(TsSchedRecord) == 16
    from paper_2604_00510_b200._abi import TsTraceRow

    assert ctypes.sizeof(TsTraceRow) == 24
    from paper_2604_00510_b200._abi import TsForest, TsSchedParams, TsTargetsInfo

    assert ctypes.sizeof(TsSchedParams) == 40
    assert ctypes.sizeof(TsTargetsInfo) == 32
    assert ctypes.sizeof(TsForest) == 8 + 11 * 8


def test_fill_problem_matches_reference_tables(lib):
    """ts_fill_problem (host code in the library) vs reference make_problem output."""
    from golden_io import load
    from paper_2604_00510_b200.backend import RewardProfile
    from paper_2604_00510_b200.engine import fill_problem

    for name in ("c1", "mixed_b3", "c4_stagnation"):
        for rec in load("workloads")[name]:
            pr = rec["profile"]
            prof = RewardProfile(tuple(pr["golden_range"]), tuple(pr["off_path_range"]), pr["hidden_until_depth"],
                                 tuple(pr["shared_range"]) if pr["shared_range"] else None, pr["target_aggregate"])
            p = fill_problem(rec["seed"], rec["golden_path"] is not None, rec["depth_range"], rec["branching"], prof)
            assert p.base_depth == rec["base_depth"]
            if rec["golden_path"] is None:
                assert p.golden_len == -1
            else:
                assert list(p.golden_path[: p.golden_len]) == rec["golden_path"]
                assert list(p.golden_rewards[: p.golden_len]) == rec["golden_rewards"]


def test_engine_fails_loudly_without_gpu(lib):
    """No CPU fallback: creating an engine on a GPU-less host is an error."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2604_00510_b200.config import SearchConfig
    from paper_2604_00510_b200.engine import Engine

    with pytest.raises(RuntimeError):
        Engine(SearchConfig(), 0)
