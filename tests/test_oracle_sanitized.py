"""The oracle under AddressSanitizer + UndefinedBehaviorSanitizer.

An out-of-bounds read in the C oracle could give right-looking numbers that the pins happen to
accept; so the same source is built with -fsanitize=address,undefined and every entry point
(every form, order 1-4, every material layout, element sub-ranges, the Stokes coupling pair,
stress, geometry, assembly, the degenerate-cell error path) runs once in a subprocess with the
sanitizer runtimes preloaded.  Any report that names the oracle fails the test.

A negative control (a heap overflow planted in a small library built and loaded the same way)
shows that the set-up detects what it is meant to; where the control cannot be made to work
(no sanitizer runtimes, or a kernel whose address-space randomisation the runtime cannot cope
with even under `setarch -R`) both tests are skipped rather than failed: that is the machine,
not the oracle."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def _runtime(name):
    p = subprocess.run(["gcc", f"-print-file-name={name}"], capture_output=True, text=True).stdout.strip()
    return p if os.path.isabs(p) and os.path.exists(p) else None


def _env():
    asan, ubsan = _runtime("libasan.so"), _runtime("libubsan.so")
    if not asan or not ubsan:
        pytest.skip("gcc sanitizer runtimes not installed")
    env = dict(os.environ)
    env.update(LD_PRELOAD=f"{asan}:{ubsan}",
               ASAN_OPTIONS="detect_leaks=0:abort_on_error=0:exitcode=87",
               UBSAN_OPTIONS="print_stacktrace=1:halt_on_error=1:exitcode=88",
               OMP_NUM_THREADS="4")
    return env


def _control(tmp_path, prefix):
    """True when the planted overflow is reported with the launch prefix `prefix`."""
    src = tmp_path / "bad.c"
    src.write_text("#include <stdlib.h>\n"
                   "double bad(int n) { double *a = malloc(n * sizeof(double)); double s = 0;\n"
                   "  for (int i = 0; i <= n; ++i) s += a[i] = i; free(a); return s; }\n")
    so = tmp_path / "libbad.so"
    subprocess.run(["gcc", "-O1", "-g", "-fsanitize=address,undefined", "-fPIC", "-shared",
                    "-o", str(so), str(src)], check=True)
    code = f"import ctypes; l = ctypes.CDLL({str(so)!r}); l.bad.restype = ctypes.c_double; l.bad(8)"
    pr = subprocess.run([*prefix, sys.executable, "-c", code], capture_output=True, text=True,
                        env=_env(), timeout=120)
    # UBSan's object-size check or ASan's redzone check, whichever fires first
    found = "heap-buffer-overflow" in pr.stderr or "runtime error:" in pr.stderr
    return pr.returncode != 0 and found and "bad.c" in pr.stderr


def _working_prefix(tmp_path):
    prefixes = [[]]
    if shutil.which("setarch"):
        prefixes.append(["setarch", os.uname().machine, "-R"])      # no address-space randomisation
    for prefix in prefixes:
        try:
            if _control(tmp_path, prefix):
                return prefix
        except (subprocess.TimeoutExpired, OSError):
            pass
    pytest.skip("the sanitizer runtimes do not work on this machine (negative control not detected)")


def test_sanitizer_setup_detects_a_planted_overflow(tmp_path):
    _working_prefix(tmp_path)       # skips when no launch prefix detects the planted overflow


def test_oracle_under_asan_ubsan(tmp_path):
    prefix = _working_prefix(tmp_path)
    env = _env()
    env["ORACLE_SANITIZE"] = "1"
    pr = subprocess.run([*prefix, sys.executable, os.path.join(HERE, "helpers", "oracle_sanitized_driver.py")],
                        capture_output=True, text=True, env=env, timeout=900)
    log = pr.stdout[-2000:] + pr.stderr[-6000:]
    assert pr.returncode == 0, log
    assert "AddressSanitizer" not in pr.stderr and "runtime error:" not in pr.stderr, log
    assert pr.stdout.strip().splitlines()[-1].startswith("done "), log
