"""The drop-in, end to end: the reference's own problem builders and run_ism (compiled from
/root/reference against oracle/eigen_shim) vs the reference-side shim run_ism_gpu
(integration/ism_gpu.cpp -> libqoc_b200.so), in one process on the B200.

The binary is built in the development container (`make -C integration`, which needs the
reference tree) and travels in-tree to the GPU box; the test is skipped where it was not built."""
import json
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
BIN = Path(__file__).resolve().parents[1] / "integration" / "_build" / "dropin_check"


@pytest.mark.skipif(not BIN.exists(), reason="integration/_build/dropin_check not built (needs /root/reference)")
def test_reference_run_ism_vs_device_dropin():
    out = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=900)
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    cases = {c["case"]: c for c in lines if "case" in c}
    for name in ("spin2_config1_200it", "spin2_direct_plan", "rotor_preset_quadratic", "condensate_preset_kat8",
                 "condensate_naive_adjoint", "monotonic_solver_rejected", "monotonic_solver_rejected_reference",
                 "spin2_monotonic", "spin2_monotonic_events", "spin2_newton", "density_matrix_spin_chain", "user_potential_plugin"):
        assert name in cases and cases[name]["ok"], (name, cases.get(name), out.stderr[-2000:])
    assert out.returncode == 0 and lines[-1] == {"all_ok": True}
