"""The C ABI from plain C (examples/c_client.c): it compiles and links against librecoil.so
with gcc (CPU), and on a GPU it encodes, combines, decodes through recoil_decoder_* with
cudaMalloc'd buffers and through recoil_multi_decode with a gather -- bit-exact."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _exe():
    from paper_2306_12141_b200 import _build
    return _build.build_c_client()


def test_c_client_builds_and_links():
    exe = _exe()
    assert os.path.exists(exe)
    out = subprocess.run(["ldd", exe], capture_output=True, text=True).stdout
    assert "librecoil.so" in out


@pytest.mark.gpu
@pytest.mark.parametrize("args", [["4000000", "1000", "0", "0"], ["777777", "64", "0", "0", "0"], ["100", "3", "0"]])
def test_c_client_decodes_bit_exact(args):
    p = subprocess.run([_exe(), *args], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "bit-exact" in p.stdout
