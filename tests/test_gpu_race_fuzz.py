"""Race check of the sweeps by schedule fuzzing (tools/race_fuzz.py).

compute-sanitizer (racecheck / memcheck) is closed on the GPU pool, so the
barrier discipline of the diagonal sweeps -- warp-pair exchange slots
double-buffered by step parity and joined by named barriers (bar.sync id, 64,
csrc/hsrq_diag_ws.cuh), the one-warp sweeps' __syncwarp column hand-offs --
the panel's cp.async pipeline and the Henry sweep's pivot exchange is checked
by perturbing the schedule instead: the `-DHSRQ_FUZZ` build sleeps random
threads for up to ~2 us after every barrier, and its outputs on solves that
take every guard path must equal the production build's bit for bit."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_schedule_fuzzed_build_is_bitwise_identical(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sys.path.insert(0, ROOT)
    from paper_2101_05063_b200 import _build

    lib = _build.variant_lib("fuzz")
    if not os.path.exists(lib) or os.path.getmtime(lib) < max(os.path.getmtime(d) for d in _build.DEPS):
        _build.build(variant="fuzz", defines=["HSRQ_FUZZ"])
    tool = os.path.join(ROOT, "tools", "race_fuzz.py")
    want = str(tmp_path / "prod.npz")
    env = {k: v for k, v in os.environ.items() if k != "HSRQ_LIB_VARIANT"}
    subprocess.run([sys.executable, tool, "--save", want], check=True, env=env, timeout=600)
    env["HSRQ_LIB_VARIANT"] = "fuzz"
    r = subprocess.run([sys.executable, tool, "--compare", want, "--reps", "2"], env=env,
                       capture_output=True, text=True, timeout=900)
    print(r.stdout, r.stderr[-2000:])
    assert r.returncode == 0, r.stdout
