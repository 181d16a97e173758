"""The reference's unit-test scenarios compiled against the C++ mirror
(include/mh/*.hpp) and run on the GPU through libmhg.so."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "dropin_test")


def test_cpp_headers_compile():
    """The C++ mirror compiles and links against libmhg.so (no GPU needed)."""
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_cpp_dropin_on_gpu(gpu):
    if not os.path.exists(BIN):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


@pytest.mark.gpu
def test_cpp_protocol_golden_csv(gpu):
    """run_trials on the GPU engine reproduces the reference's 20-trial golden
    CSV (bench_test.cpp:528-549, time columns stripped); io round trip."""
    exe = os.path.join(ROOT, "tests", "cpp", "protocol_test")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    golden = os.path.join(ROOT, "tests", "golden", "bench_trials_seed0_n64_t8_q2.csv")
    r = subprocess.run([exe, golden], capture_output=True, text=True, timeout=300, cwd="/tmp")
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("n,t,q", [(64, 8, 97), (24, 3, 2), (256, 32, 65521), (128, 64, 2147483647)])
def test_cpp_save_matrix_bytes_equal_reference(gpu, tmp_path, n, t, q):
    """io.hpp:16-26: the mirror's save_matrix_file (device Morton -> row-major kernel)
    writes byte-for-byte the file the reference's writer (oracle/_ref) writes for the
    same mh::Rng(seed) container; the mirror loads it back exactly."""
    from oracle.binding import REF_SO, Reference
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref/libmhref.so not built")
    exe = os.path.join(ROOT, "tests", "cpp", "protocol_test")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    ours, ref = tmp_path / "ours.txt", tmp_path / "ref.txt"
    r = subprocess.run([exe, "--save", str(n), str(t), str(q), "5", str(ours)], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    Reference().save_matrix(n, t, q, 5, str(ref))
    assert ours.read_bytes() == ref.read_bytes()
