"""C-ABI surface checks that need no GPU: libqoc_b200.so loads, exports every entry point that
include/qoc_gpu.h declares, and the ctypes mirror matches the header's struct layout."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1603_01237_b200 import _native, abi
from paper_1603_01237_b200 import ism as I
from tests import oracle_api as O

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "qoc_gpu.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int32_t|int64_t|void|const char\*)\s+(qoc_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("qoc_ism_run", "qoc_ctx_create", "qoc_ctx_destroy", "qoc_propagate_final",
                 "qoc_objective_gradient", "qoc_assemble_propagator"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _native.lib()  # loads libqoc_b200.so (built by __graft_entry__.build)
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.qoc_abi_version() == abi.QOC_ABI_VERSION


def test_oracle_is_a_separate_library():
    # the product library must not contain the checker
    data = _native.LIB_PATH.read_bytes()
    assert b"oracle_ism_run" not in data
    assert hasattr(O.lib(), "oracle_ism_run")


def test_struct_layout_matches_header_sizes():
    # the header's structs are plain C; compile a tiny probe with gcc and compare sizeof/offsetof
    import subprocess
    import tempfile
    probe = r'''
#include <stdio.h>
#include <stddef.h>
#include "qoc_gpu.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu\n", sizeof(qoc_problem_v1), sizeof(qoc_ism_config_v1),
         sizeof(qoc_solver_v1), sizeof(qoc_iter_record_v1), sizeof(qoc_run_status_v1),
         sizeof(qoc_profile_v1), sizeof(qoc_ctx_opts_v1));
  printf("%zu %zu %zu\n", offsetof(qoc_problem_v1, initial), offsetof(qoc_problem_v1, kappa),
         offsetof(qoc_ism_config_v1, node_index));
  return 0;
}
'''
    with tempfile.TemporaryDirectory() as td:
        src = Path(td) / "p.c"
        src.write_text(probe)
        exe = Path(td) / "p"
        subprocess.run(["gcc", "-I", str(ROOT / "include"), "-o", str(exe), str(src)], check=True)
        out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()
    sizes = [int(v) for v in out]
    mine = [C.sizeof(abi.ProblemV1), C.sizeof(abi.IsmConfigV1), C.sizeof(abi.SolverV1),
            C.sizeof(abi.IterRecordV1), C.sizeof(abi.RunStatusV1), C.sizeof(abi.ProfileV1),
            C.sizeof(abi.CtxOptsV1), abi.ProblemV1.initial.offset, abi.ProblemV1.kappa.offset,
            abi.IsmConfigV1.node_index.offset]
    assert sizes == mine


def test_context_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(Exception):
        _native.Context()


def test_balanced_partition():
    assert I.balanced_nodes(20000, 128)[:3] == [0, 157, 314]
    lens = np.diff(I.balanced_nodes(20000, 128))
    assert lens.sum() == 20000 and (lens == 157).sum() == 32 and (lens == 156).sum() == 96
    lens = np.diff(I.balanced_nodes(4000, 256))
    assert (lens == 16).sum() == 160 and (lens == 15).sum() == 96
    assert I.balanced_nodes(1000, 8) == list(range(0, 1001, 125))


def test_control_layout_round_trip():
    u = np.arange(2 * 5 * 3, dtype=np.float64).reshape(2, 3, 5)  # (B, C, K)
    flat = I.controls_to_abi(u, 2, 3, 5)
    # column-major C x K per problem: (c, j) at c + j*C (controls.hpp:54)
    assert flat[1 * 15 + 2 + 4 * 3] == u[1, 2, 4]
    assert np.array_equal(I.controls_from_abi(flat, 2, 3, 5), u)
