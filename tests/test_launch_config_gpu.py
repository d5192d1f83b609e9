"""Launch-configuration invariance: a copy of libmem built
with other CTA sizes and work splits -- k_points items of 64 points instead of 128, k_bin CTAs
of 128 threads (tiles of 1024 points), k_sort CTAs of 128 threads, k_fuse CTAs of 256 threads, k_refold CTAs of
256 threads (sorted lists of up to 8192 points), k_smap CTAs of 512 threads, k_image CTAs of
128 threads with 8 lanes per cell, one-map RED passes in cell waves of a 1 MB scratch -- must produce exactly the bits of the shipped library on
every point path, the image pass and the PCA readout (tests/launch_variant_run.py)."""
import os
import shutil
import subprocess
import sys
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2309_16818_b200"))

VARIANT = ["MEM_WARP_PTS=2", "MEM_BIN_THREADS=128", "MEM_SORT_THREADS=128", "MEM_FUSE_THREADS=256",
           "MEM_REFOLD_THREADS=256", "MEM_SMAP_THREADS=512", "MEM_IMG_THREADS=128", "MEM_IMG_LANES=8",
           "MEM_CELL_WAVE_MB=1"]


@pytest.mark.gpu
def test_other_launch_configurations_give_identical_bits():
    import build  # paper_2309_16818_b200/build.py
    if not os.path.exists(build.NVCC) and shutil.which("nvcc") is None:
        pytest.skip("nvcc not available")
    tmp = tempfile.mkdtemp()
    lib = build.build_variant(os.path.join(tmp, "libmem_variant.so"), VARIANT)
    runs = []
    for env_lib in (None, lib):
        env = dict(os.environ)
        env.pop("MEM_LIB", None)
        if env_lib:
            env["MEM_LIB"] = env_lib
        out = os.path.join(tmp, f"run{len(runs)}.npz")
        subprocess.run([sys.executable, os.path.join(ROOT, "tests", "launch_variant_run.py"), out], env=env,
                       check=True, timeout=900)
        runs.append(np.load(out))
    a, b = runs
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        assert np.array_equal(a[k], b[k], equal_nan=True), k
    shutil.rmtree(tmp, ignore_errors=True)
