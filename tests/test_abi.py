"""CPU: the C ABI boundary (include/kvlinc.h <-> libkvlinc.so <-> ctypes).

No compute calls need a GPU here: the library must load, export every symbol
the header declares, agree with the ctypes struct layouts, and refuse to
compute without an sm_100 device (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2510_05373_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "kvlinc.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(kvlc_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.EXPORTED), set(names) ^ set(_lib.EXPORTED)
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (kvlc_[a-z0-9_]+)", out))
    assert set(names) <= exported


def test_struct_layouts_match_header(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(f'''#include <stdio.h>
#include <stddef.h>
#include "{HEADER}"
int main(void) {{
  printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(kvlc_cache), offsetof(kvlc_cache, kcodes),
         offsetof(kvlc_cache, res_len), sizeof(kvlc_adapter), offsetof(kvlc_adapter, enabled),
         sizeof(kvlc_decode_opts));
  return 0;
}}''')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(_lib.KvlcCache), _lib.KvlcCache.kcodes.offset, _lib.KvlcCache.res_len.offset,
            ctypes.sizeof(_lib.KvlcAdapter), _lib.KvlcAdapter.enabled.offset,
            ctypes.sizeof(_lib.KvlcDecodeOpts)]
    assert got == want


def test_constants_match_header():
    text = open(HEADER).read()
    consts = dict(re.findall(r"#define (KVLC_\w+) (\d+)", text))
    assert int(consts["KVLC_D"]) == _lib.D and int(consts["KVLC_G"]) == _lib.G
    assert int(consts["KVLC_R"]) == _lib.R and int(consts["KVLC_RANK"]) == _lib.RANK
    assert int(consts["KVLC_SLOTS"]) == _lib.SLOTS
    assert int(consts["KVLC_EINVAL"]) == _lib.KVLC_EINVAL and int(consts["KVLC_ENODEV"]) == _lib.KVLC_ENODEV


def test_version_and_sizes_without_device():
    lib = _lib.load()
    assert lib.kvlc_version() >= 10000
    assert lib.kvlc_ref_flush_scratch(128, 128, 256) > 128 * 128 * 8
    assert lib.kvlc_ref_decode_scratch(64, 4096, 128, 32, 32) > 0


@pytest.mark.skipif(_lib.device_ok(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    """Every compute entry point refuses to run without an sm_100 GPU."""
    lib = _lib.load()
    assert lib.kvlc_device_ok() == 0
    rc = lib.kvlc_ref_pack(None, 1, 1, 2, None, None)
    assert rc == _lib.KVLC_ENODEV and "no CPU path" in _lib.last_error()
    rc = lib.kvlc_decode(None, None, None, None, None, None, 0, None)
    assert rc == _lib.KVLC_ENODEV
    import numpy as np
    import paper_2510_05373_b200 as qk
    with pytest.raises(_lib.KvlcError, match="no CPU fallback"):
        qk.pack_codes(np.array([1, 2, 3]), 2)
    with pytest.raises(_lib.KvlcError):
        qk.quantize_tensor(np.ones((4, 4)), qk.QuantConfig())
    from paper_2510_05373_b200.batched import BatchedKVCache
    with pytest.raises(_lib.KvlcError):
        BatchedKVCache(1, 1, 4, 256)
