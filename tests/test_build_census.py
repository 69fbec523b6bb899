"""The serial engine's compiled form in the in-tree library (CPU only).

ptxas allocates the serial engine's out-of-line functions together with each
kernel body; an unrelated edit can make se::walk spill or flip se::w32 to its
uniform-datapath form (profiles/r02/ab_upper_band.txt: 4-13 %
on every config).  The bench numbers were measured on the form checked here."""
import os
import shutil

import pytest

from paper_1204_5882_b200 import build as B


@pytest.fixture(scope="module")
def cen():
    if not os.path.exists(B.OUT):
        pytest.skip("libpolarsc.so is not built")
    if not (shutil.which("cuobjdump") and shutil.which("nvdisasm")):
        pytest.skip("cuobjdump / nvdisasm not on PATH")
    return B.census()


def test_production_kernels_present(cen):
    for name, d in cen.items():
        assert d["body"] > 1000 and d["w32"] > 100 and d["walk"] > 100, (name, d)


def test_serial_engine_does_not_spill(cen):
    for name, d in cen.items():
        assert d["walk_stl"] == 0 and d["w32_stl"] == 0, (name, d)


def test_bench_kernels_w32_is_the_vector_form(cen):
    # c2-c4 run the unclustered kernel, c5 the 512-thread kernel with K = 4 compiled in
    for name in ("unclustered", "clustered512_k2", "clustered512_k4", "clustered512_k8"):
        assert cen[name]["w32_r2ur"] == 0, (name, cen[name])
