"""The fp32 branch-free math of the stage-2 kernels against the routines it replaces, on the
device (csrc/common.cuh atan2_nobranch, csrc/stage2.cuh wrap_yaw / np_mod_pos folds):
bit-for-bit over 2^24 pseudo-random inputs, including zeros, infinities and NaNs."""
import numpy as np
import pytest

from paper_2510_07674_b200 import _native as nat

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [1, 12345])
def test_branch_free_math_is_bitwise_equal(seed):
    lib = nat.load()
    counts = np.zeros(3, dtype=np.int64)
    assert lib.spasm_selftest_math(1 << 24, seed, counts.ctypes.data) == 0
    assert counts.tolist() == [0, 0, 0]
