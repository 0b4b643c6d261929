"""GPU: frames and depth sorts in flight on several contexts at once.

Round 1 saw intermittent wrong depth orders only when several liblodge
contexts rendered concurrently.  The cause was a warp left diverged by the
per-lane look-back spin of the onesweep partition reaching an aligned CTA
barrier (csrc/onesweep.cuh);
a library rebuilt without the reconvergence (-DLODGE_OS_NO_RECONVERGE) still
fails these stresses within seconds (profiles/r02_stress.md).

* the depth sort alone (lodge_debug_depth_sort) on 4 and 8 streams, every
  result against torch's stable sort of the same keys (np.lexsort((index,
  depth)), reference src/raster.py:401);
* whole config-3 frames, 4 slots, 27 x 16 views spread over the sweep: every
  frame's outputs (image, per_pixel_visible, per_tile_count, max weights)
  bit-identical to the same view rendered serially on one stream, and -- in
  a LODGE_VERIFY build, in a subprocess -- the device order checks of the
  depth sort, every staged onesweep partition, every per-tile list and
  every block list (order, masks, per-tile counts) silent.
"""

import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.mark.parametrize("streams,rounds", [(4, 1500), (8, 750)])
def test_depth_sort_concurrent_contexts(streams, rounds):
    from tests import stress_sort
    res = stress_sort.run(streams=streams, n=1_600_000, rounds=rounds, seed=streams)
    assert res["sorts"] == streams * rounds
    assert res["bad"] == 0, res
    assert not res["fault_bits"], res


def test_frames_in_flight_bitwise():
    from tests import stress_frames
    res = stress_frames.run("config3", streams=4, frames=432, reps=2, seed_views=11)
    assert res["frames"] == 864
    assert res["output_mismatch"] == 0, res
    assert not res["fault_frames"] and res["sticky"] == 0, res
    assert res["overflow"] == 0


def _verify_lib():
    from paper_2505_23158_b200 import _native
    _native.build()  # make: brings the diagnostic variants up to date with the sources
    return os.path.join(os.path.dirname(_native.LIB_PATH), "liblodge_verify.so")


def test_frames_in_flight_verify_build():
    """LODGE_VERIFY: depth order after the sort, every onesweep partition's
    staging, every per-tile list after each tile sort, checked on the device
    for every frame (FAULT_DEPTH / FAULT_STAGE / FAULT_LISTORD)."""
    assert os.path.exists(_verify_lib())
    env = dict(os.environ, LODGE_LIB="verify")
    out = subprocess.run([sys.executable, "-m", "tests.stress_frames", "--config", "config3",
                          "--streams", "4", "--frames", "432", "--reps", "3", "--seed", "12"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["lib"] == "verify" and res["frames"] == 1296
    assert res["output_mismatch"] == 0, res
    assert not res["fault_frames"] and res["sticky"] == 0, res
