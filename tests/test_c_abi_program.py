"""The boundary is a real C ABI: a plain C program (examples/c_abi_gather.c) that includes only
include/dgz.h and links libdgz.so samples a minibatch on the GPU, gathers it by zero-copy and
memcmp-checks every row against the host table."""
import os
import subprocess

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "examples", "c_abi_gather")


def _build():
    from paper_2103_03330_b200 import build
    build.build()
    assert os.path.exists(BIN)


def test_c_program_links_against_the_abi():
    _build()
    out = subprocess.run(["nm", "-u", BIN], capture_output=True, text=True).stdout
    assert "dgz_gather_perm" in out and "dgz_sample_uniform" in out and "torch" not in out


@pytest.mark.gpu
@pytest.mark.parametrize("rows,dim", [(20000, 100), (5000, 602), (300, 128)])
def test_c_program_bit_exact(rows, dim):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _build()
    r = subprocess.run([BIN, str(rows), str(dim)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 mismatches" in r.stdout
