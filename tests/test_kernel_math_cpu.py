"""The kernels' per-thread arithmetic, pinned on the CPU (no GPU needed).

`tests/emu/kernel_math_emu.cpp` compiles the product's own device arithmetic
(`paper_2111_08692_b200/csrc/utf8.cuh`, `utf16.cuh`, host-compilable through `swar.cuh`) with
g++ and runs it in the kernels' lane / warp / tile layout -- 32-byte thread chunks, 1 KiB
warps, the ASCII-warp skip, the classifier's 3-byte look-ahead in the last lane of EVERY warp,
the exact rescan of flagged warps -- against the oracle (oracle/oracle.c), which shares no
code with it.  What it pins (D2-D5):

* the bit-plane classifier `u8::analyze32` (the one the kernels run): on every string of
  length <= 4 over the 27-byte class alphabet, at every phase of a 32-byte chunk and across
  a warp (= tile) edge, followed by text or ending the input, valid input never flags and the
  first flag r of invalid input obeys e <= r <= e + 3 in the warp that owns e; the rescan
  (`u8::err_at`) of the flagged warps returns exactly the oracle's first error e;
* the end-position decoder `u8::units4` and its emit mask (equal to the classifier's) on
  random config-0 text, corrupted / truncated copies and byte soup at input alignments
  0 / 1 / 7 / 15: the staged units equal the oracle's output on [0, written);
* `u8::units4_nof` (f1 for UTF-8): on every warp with no >= F0 lead in its 1 KiB or the 3 bytes
  before, the same emit mask and units as `u8::units4`;
* the f4 keyed 12-byte decoder (`keyed::decode_thread`, utf8_keyed.cuh, with the library's
  own tables) on the same chunks and on width-dense text (one width, or any subset of the
  four): its units, at the same per-thread slots, equal the oracle's on [0, written), and on
  valid input it emits exactly the thread's count;
* the UTF-8 plan's arithmetic (`u8::plan_weight`, `u8::pending3`): at every cut of random,
  corrupted and soup text, equal to the emit count (`u8::emits_at`) up to the first error and
  never below the units written before it past the error;
* the UTF-16 -> UTF-8 byte-SWAR (`u16::classes4 / widths / encode4`, pairing predicate):
  first error, per-thread counts and staged bytes against the oracle.
"""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "emu", "kernel_math_emu.cpp")


@pytest.fixture(scope="module")
def emu(tmp_path_factory):
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("g++ not available")
    exe = str(tmp_path_factory.mktemp("emu") / "kernel_math_emu")
    subprocess.check_call([gxx, "-O2", "-std=c++17",
                           "-I" + os.path.join(ROOT, "paper_2111_08692_b200", "csrc"),
                           "-o", exe, SRC, os.path.join(ROOT, "oracle", "oracle.c")])
    return exe


def _run_parallel(cmds, timeout=900):
    procs = [subprocess.Popen(c, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for c in cmds]
    outs = []
    for p in procs:
        out, _ = p.communicate(timeout=timeout)
        outs.append((p.returncode, out))
    return outs


def test_bitplane_window_exhaustive_alphabet(emu):
    """551,881 strings x 42 placements x {followed by text, ending the input}."""
    parts = max(1, min(16, os.cpu_count() or 1))
    outs = _run_parallel([[emu, "window8", str(k), str(parts)] for k in range(parts)])
    cases = 0
    for rc, out in outs:
        assert rc == 0, out
        cases += int(out.split(":")[1].split("cases")[0])
    assert cases == 551881 * 42 * 2, cases


def test_utf8_decode_layout_fuzz(emu):
    out = subprocess.run([emu, "fuzz8", "400"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout


def test_utf16_encode_layout_fuzz(emu):
    out = subprocess.run([emu, "fuzz16", "600"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout


def test_plan_arithmetic_every_cut(emu):
    """The UTF-8 plan (length formula + pending units at the cuts, kernels.cu k_plan8) equals
    the kernel's emit count at every cut up to the first error and never falls below the units
    written before it past the error ("planned")."""
    out = subprocess.run([emu, "plan8", "3000"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout


def test_keyed_fast_paths_build(tmp_path):
    """The f4 decoder with the paper's three homogeneous fast paths (-DUG_KEYED_FASTPATHS,
    PAPER.md:96; off in the default build) against the oracle on the same fuzz."""
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("g++ not available")
    exe = str(tmp_path / "emu_fp")
    subprocess.check_call([gxx, "-O2", "-std=c++17", "-DUG_KEYED_FASTPATHS",
                           "-I" + os.path.join(ROOT, "paper_2111_08692_b200", "csrc"),
                           "-o", exe, SRC, os.path.join(ROOT, "oracle", "oracle.c")])
    out = subprocess.run([exe, "fuzz8", "300"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout
