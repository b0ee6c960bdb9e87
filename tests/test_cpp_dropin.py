"""The C++ drop-in boundary (include/efta_b200.hpp) has a real C++ consumer:
tests/cpp/acceptance_gpu.cpp re-runs the reference's acceptance checks 1, 2, 4 (d = 64 and 128),
7 and 10, the ABFT operator API (encode_strided / checksummed_gemm / verify_locate_correct) and the
decoupled baseline (decoupled_ft_forward)
through efta_b200:: on the GPU. CPU: it compiles and links against libefta_b200.so. GPU: every
check passes."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "acceptance_gpu")


def _build():
    r = subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp"), "-s"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert os.path.exists(BIN)


def test_cpp_consumer_compiles_and_links():
    _build()


@pytest.mark.gpu
def test_cpp_acceptance_checks_pass_on_gpu():
    _build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=1200)
    lines = [x for x in r.stdout.splitlines() if x.startswith("[")]
    out = os.environ.get("EFTA_PARITY_OUT")
    if out:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, "cpp_acceptance.txt"), "w") as f:
            f.write(r.stdout + r.stderr)
    assert len(lines) == 8, r.stdout + r.stderr
    assert r.returncode == 0 and all(x.startswith("[PASS]") for x in lines), "\n".join(lines) + r.stderr
