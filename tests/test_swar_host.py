"""Host check of the byte-plane SWAR arithmetic of the UTF-16 -> UTF-8 kernel.

csrc/vt_swar.cuh compiles for the host with LOP3 / PRMT emulated bit-exactly;
tests/swar_host/u16_planes_test.cpp runs the same plane functions the kernel
runs over every BMP unit in every lane, every surrogate half, pairs cut by a
range start, long valid streams (against a plain UTF-8 encoder, the layout of
proj/src/codec_core.cpp:60-72) and the pairing / count planes on arbitrary
windows (against the scalar pairing rule, proj/src/codec_core.cpp:106-125).
No GPU needed.
"""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_u16_planes_host(tmp_path):
    exe = str(tmp_path / "u16_planes_test")
    src = os.path.join(ROOT, "tests", "swar_host", "u16_planes_test.cpp")
    subprocess.run(["g++", "-O2", "-std=c++17", "-x", "c++", src, "-o", exe], check=True)
    out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    assert out.startswith("OK "), out
    assert int(out.split()[1]) > 900000
