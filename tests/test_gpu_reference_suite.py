"""The reference's own unit tests (pkg/tests/test_{quantize,hadamard,cache,attention}.py),
run unchanged against this package imported as `quantkv` (the drop-in claim).

The four files travel as tests/golden/reftests.tar.gz (made by
tests/golden/make_reftests.py from /root/reference, checksums in
reftests.sha256).  They are extracted into a temporary directory next to a
conftest.py that registers `quantkv` and its submodules as aliases of
paper_2510_05373_b200, and run by pytest in a subprocess.  Every compute call
goes through libkvlinc.so (the shim has no CPU path), so this needs the GPU.
"""
import hashlib
import os
import subprocess
import sys
import tarfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")

ALIAS = '''import sys
sys.path.insert(0, {root!r})
import paper_2510_05373_b200 as pkg
from paper_2510_05373_b200 import adapter, attention, cache, hadamard, linalg, quantize
sys.modules["quantkv"] = pkg
for name, mod in (("adapter", adapter), ("attention", attention), ("cache", cache),
                  ("hadamard", hadamard), ("linalg", linalg), ("quantize", quantize)):
    sys.modules["quantkv." + name] = mod
'''


def _extract(dst):
    want = dict(line.split()[::-1] for line in open(os.path.join(GOLDEN, "reftests.sha256")) if line.strip())
    with tarfile.open(os.path.join(GOLDEN, "reftests.tar.gz")) as tar:
        for m in tar.getmembers():
            data = tar.extractfile(m).read()
            assert hashlib.sha256(data).hexdigest() == want[m.name], m.name
            with open(os.path.join(dst, m.name), "wb") as fh:
                fh.write(data)
    (dst / "conftest.py").write_text(ALIAS.format(root=ROOT))
    return sorted(want)


def _run(tmp_path, *extra):
    files = _extract(tmp_path)
    return subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir",
                           str(tmp_path), *extra, *[str(tmp_path / f) for f in files]],
                          capture_output=True, text=True, cwd=tmp_path, timeout=1800)


def test_reference_unit_tests_collect_against_the_shim(tmp_path):
    """CPU: the archive matches its checksums and every reference test imports and collects
    against the shim's names (65 tests)."""
    r = _run(tmp_path, "--collect-only")
    tail = r.stdout.strip().splitlines()[-3:]
    assert r.returncode == 0, r.stdout[-3000:]
    assert "65 tests collected" in tail[-1], tail


@pytest.mark.gpu
def test_reference_unit_tests_pass_against_the_shim(tmp_path):
    r = _run(tmp_path)
    tail = r.stdout.strip().splitlines()[-15:]
    print("\n".join(tail))
    assert r.returncode == 0, "\n".join(tail)
    assert " passed" in tail[-1] and "failed" not in tail[-1] and "error" not in tail[-1]
