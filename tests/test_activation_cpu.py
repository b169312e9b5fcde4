"""Host-side activation and sharding invariants (paper_2509_26581_b200/csrc/
activate.cpp), compiled with AddressSanitizer: tile/slot/partial-plan
consistency, 8-edge padding, local camera lists, and that shards partition
points and edges exactly."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2509_26581_b200", "csrc")


def test_activation_invariants_asan(tmp_path):
    exe = str(tmp_path / "activation_test")
    subprocess.check_call(["g++", "-std=c++17", "-O1", "-g", "-fsanitize=address,undefined", "-I", CSRC, "-I",
                           os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "cpp", "activation_test.cpp"),
                           os.path.join(CSRC, "activate.cpp"), os.path.join(CSRC, "synth.cpp"), "-o", exe])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "activation invariants ok" in out.stdout
