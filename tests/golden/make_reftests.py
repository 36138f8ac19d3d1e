"""Package the reference's own unit tests for the hot path as a test fixture.

    python tests/golden/make_reftests.py

Reads /root/reference/pkg/tests/test_{quantize,hadamard,cache,attention}.py
(present only in the build container) and writes them, unmodified, into
tests/golden/reftests.tar.gz with their sha256 in tests/golden/reftests.sha256.
tests/test_gpu_reference_suite.py extracts the archive on the GPU box and runs
the files with pytest against this package imported under the name `quantkv`
(the drop-in claim of INTEGRATION.md).  The archive is a fixture, like the
.npz golden vectors: nothing in the product imports it.
"""
import hashlib
import io
import os
import tarfile

SRC = "/root/reference/pkg/tests"
FILES = ("test_quantize.py", "test_hadamard.py", "test_cache.py", "test_attention.py")
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    buf = io.BytesIO()
    sums = []
    with tarfile.open(fileobj=buf, mode="w:gz") as tar:
        for f in FILES:
            data = open(os.path.join(SRC, f), "rb").read()
            info = tarfile.TarInfo(f)
            info.size, info.mtime, info.mode = len(data), 0, 0o644
            tar.addfile(info, io.BytesIO(data))
            sums.append(f"{hashlib.sha256(data).hexdigest()}  {f}")
    with open(os.path.join(HERE, "reftests.tar.gz"), "wb") as fh:
        fh.write(buf.getvalue())
    with open(os.path.join(HERE, "reftests.sha256"), "w") as fh:
        fh.write("\n".join(sums) + "\n")
    print("\n".join(sums))


if __name__ == "__main__":
    main()
