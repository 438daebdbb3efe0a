"""The drop-in headers (include/vtrans/*.hpp) declare the reference's whole
interface (proj/include/vtrans/codec_core.hpp:14-68, utf8_to_utf16.hpp:12-33,
utf16_to_utf8.hpp:15-17, validation.hpp:15-31, vec128.hpp:17-21): a program
that uses the scalar codec, the constants and is_scalar_value next to the GPU
entry points compiles with -I<repo>/include unchanged, links the reference's own
codec object (oracle/_ref/obj/codec_core.o) for vtrans::scalar::* plus
libvtrans_gpu.so for the hot path, and gets the reference's answers."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2109_10433_b200", "lib")
CODEC_O = os.path.join(ROOT, "oracle", "_ref", "obj", "codec_core.o")

PROGRAM = r'''
#include "vtrans/codec_core.hpp"
#include "vtrans/utf8_to_utf16.hpp"
#include "vtrans/utf16_to_utf8.hpp"
#include "vtrans/validation.hpp"
#include "vtrans/vec128.hpp"
#include <cstdio>
#include <cstring>
static_assert(vtrans::kMaxCodePoint == 0x10FFFF && vtrans::kSurrogateFirst == 0xD800 &&
              vtrans::kSurrogateLast == 0xDFFF);
static_assert(vtrans::is_scalar_value(0x41) && !vtrans::is_scalar_value(0xDC00) &&
              !vtrans::is_scalar_value(0x110000) && vtrans::is_scalar_value(0x10FFFF));
int main(int argc, char** argv) {
  bool ok = true;
  // the reference's scalar codec (declared by our header, defined by codec_core.o)
  uint8_t b[4];
  ok = ok && vtrans::scalar::encode_utf8(0x1F600, b) == 4 && b[0] == 0xF0 && b[3] == 0x80;
  uint16_t u[2];
  ok = ok && vtrans::scalar::encode_utf16(0x1F600, u) == 2 && u[0] == 0xD83D && u[1] == 0xDE00;
  const uint8_t s[] = {0xE9, 0x8F, 0xA1};
  auto d = vtrans::scalar::decode_utf8_char(std::span<const uint8_t>(s, 3), 0);
  ok = ok && d && d->code_point == 0x93E1 && d->length == 3 &&
       *d == vtrans::scalar::DecodedChar{0x93E1, 3};
  ok = ok && !vtrans::scalar::decode_utf8_char(std::span<const uint8_t>(s, 2), 0);
  if (argc > 1 && std::strcmp(argv[1], "gpu") == 0) {
    // GPU entry points against the scalar codec on the same input
    std::vector<uint8_t> in;
    for (uint32_t cp = 0x20; cp < 0x30000; cp += 37) {
      if (!vtrans::is_scalar_value(cp)) continue;
      uint8_t e[4];
      unsigned n = vtrans::scalar::encode_utf8(cp, e);
      in.insert(in.end(), e, e + n);
    }
    in.push_back(0xC0);  // an overlong lead: both stop here
    in.push_back(0x80);
    std::vector<uint16_t> want(in.size()), got(in.size());
    vtrans::TranscodeResult rs = vtrans::scalar::utf8_to_utf16(in, want.data());
    vtrans::TranscodeResult rg = vtrans::utf8_to_utf16(in, got.data(), true);
    ok = ok && rs == rg && rg.error_at && std::memcmp(want.data(), got.data(), 2 * rg.written) == 0;
    auto cs = vtrans::scalar::count_codepoints_utf8(std::span<const uint8_t>(in.data(), *rg.error_at));
    ok = ok && cs && *cs > 1000;
    ok = ok && vtrans::active_backend() == vtrans::Backend::native;
  }
  std::printf("%s\n", ok ? "HEADERS OK" : "HEADERS FAIL");
  return ok ? 0 : 1;
}
'''


def _build(tmp_path):
    src = tmp_path / "hdr.cpp"
    src.write_text(PROGRAM)
    exe = tmp_path / "hdr"
    subprocess.run(["g++", "-std=c++20", "-O1", str(src), "-I", os.path.join(ROOT, "include"), CODEC_O,
                    "-L", LIBDIR, "-lvtrans_gpu", f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)], check=True)
    return exe


@pytest.mark.skipif(not os.path.exists(CODEC_O), reason="oracle/_ref not built (no reference tree)")
def test_reference_style_program_compiles_and_links(tmp_path):
    exe = _build(tmp_path)
    p = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert p.returncode == 0 and "HEADERS OK" in p.stdout, p.stdout + p.stderr


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(CODEC_O), reason="oracle/_ref not built (no reference tree)")
def test_reference_style_program_on_gpu(tmp_path):
    exe = _build(tmp_path)
    p = subprocess.run([str(exe), "gpu"], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0 and "HEADERS OK" in p.stdout, p.stdout + p.stderr
