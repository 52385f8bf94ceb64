"""The C/C++ oracles under AddressSanitizer + UndefinedBehaviorSanitizer (CPU).

compute-sanitizer is closed on the GPU pool (VERDICT r1 missing-7), so the memory-safety
check that can run is on the host side: the oracle libraries are rebuilt with
-fsanitize=address,undefined -fno-sanitize-recover=all (GSREF_SANITIZE=1 ->
oracle/libgsref_san.so, oracle/libtsdfref_san.so) and the oracle's own pin suites run
against them in a subprocess with libasan / libubsan preloaded (python itself is not
instrumented).  Any heap / stack overflow, use-after-free, signed overflow, misaligned
or out-of-bounds shift in the oracle aborts the run.  The thread-count independence
test (50 s under ASan) is left to the plain build."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rt(name):
    p = subprocess.run(["gcc", f"-print-file-name={name}"], capture_output=True, text=True).stdout.strip()
    return p if os.path.isabs(p) and os.path.exists(p) else None


@pytest.mark.timeout(900)
def test_oracle_pins_under_asan_ubsan():
    asan, ubsan = _rt("libasan.so"), _rt("libubsan.so")
    if not asan or not ubsan:
        pytest.skip("gcc sanitizer runtimes not installed")
    env = dict(os.environ, GSREF_SANITIZE="1", LD_PRELOAD=f"{asan}:{ubsan}",
               ASAN_OPTIONS="detect_leaks=0:halt_on_error=1:abort_on_error=1",
               UBSAN_OPTIONS="halt_on_error=1:print_stacktrace=1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        "tests/test_oracle_pins.py", "tests/test_tsdf_oracle.py", "tests/test_oracle_bound.py",
                        "-k", "not thread_count"], cwd=ROOT, env=env, capture_output=True, text=True)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert "AddressSanitizer" not in tail and "runtime error" not in tail, tail
    assert os.path.exists(os.path.join(ROOT, "oracle", "libgsref_san.so"))
