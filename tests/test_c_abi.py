"""The C ABI is usable from plain C, without the Python package:
examples/c_abi_eval.c packs the reference's worked example with
rcpsp_pack_instance, evaluates it with rcpsp_eval_batch (makespan 22, the
reference's starts, test_evaluator.py:196-201) and runs one chunk with
rcpsp_run_chunk_batch.  CPU: it compiles and links against the header and
the library; GPU: it runs and checks its results."""

import shutil
import subprocess

import pytest

from conftest import ROOT, gpu_available

LIB = ROOT / "paper_1711_04556_b200" / "_lib"


def _build(tmp_path):
    if shutil.which("gcc") is None or not (LIB / "libb200tabu.so").exists():
        pytest.skip("gcc or the library missing")
    exe = tmp_path / "c_abi_eval"
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-I", str(ROOT / "include"),
           "-I", "/usr/local/cuda/include", str(ROOT / "examples" / "c_abi_eval.c"),
           "-o", str(exe), "-L", str(LIB), "-lb200tabu", "-L", "/usr/local/cuda/lib64",
           "-lcudart", f"-Wl,-rpath,{LIB}", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_example_compiles(tmp_path):
    _build(tmp_path)


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    if not gpu_available():
        pytest.skip("no GPU")
    exe = _build(tmp_path)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "cpm 16" in out.stdout
    assert "cmax 22 err 0 starts 0 0 4 4 7 12 9 12 20 15 16 22 -> ok" in out.stdout
