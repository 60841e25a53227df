"""The CPU oracle under AddressSanitizer + UndefinedBehaviorSanitizer: every entry
point of oracle/oracle.h on a small two-slab pair (tests/c/oracle_sanitize.c), including its
closed-form checks; any sanitizer report aborts the program."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_oracle_clean_under_asan_ubsan(tmp_path):
    exe = str(tmp_path / "oracle_sanitize")
    subprocess.run(["gcc", "-std=c99", "-O1", "-g", "-fno-omit-frame-pointer", "-fsanitize=address,undefined",
                    "-fno-sanitize-recover=all", "-Wall", "-Werror", "-I" + os.path.join(ROOT, "oracle"),
                    "-I" + os.path.join(ROOT, "tests", "c"), os.path.join(ROOT, "oracle", "oracle.c"),
                    os.path.join(ROOT, "tests", "c", "oracle_sanitize.c"), "-lm", "-o", exe],
                   check=True, capture_output=True, text=True)
    env = dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=1", UBSAN_OPTIONS="halt_on_error=1")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "oracle_sanitize ok" in r.stdout
