"""No C++ exception crosses the C ABI (include/pspmm.h, "Errors"; SURVEY
§8(b)): a crafted PCSR file header is rejected before any header-sized
allocation, a host allocation failure inside an entry comes back as
PSPMM_ERR_OOM instead of std::terminate, and every status-returning
extern "C" definition runs its body through pspmm::guarded.  CPU only."""
import os
import re
import struct
import subprocess
import sys
import textwrap

import pytest

from conftest import ROOT

CSRC = os.path.join(ROOT, "paper_2605_15695_b200", "csrc")


def _header(n, P, nv, V, S, omega, units, sg, nnz, ncols):
    return (b"PCSR" + struct.pack("<I", 1) + struct.pack("<QQQ", n, P, nv) +
            struct.pack("<BBH", V, S, omega) + struct.pack("<I", 0) +
            struct.pack("<QQQQ", units, sg, nnz, ncols))


@pytest.mark.parametrize("units,nv,S", [(2**31 - 2, 0, 1), (1000, 2**31 - 2, 0)])
def test_crafted_header_rejected_without_allocation(tmp_path, units, nv, S):
    from paper_2605_15695_b200 import api
    n = 1000
    p = tmp_path / "crafted.pcsr"
    # a header claiming ~2^31 chunks (or vectors) with no arrays behind it:
    # the size check fires before anything is allocated from the header
    p.write_bytes(_header(n, n, nv, 1, S, 32, units, 1 if S else 0, 0, n))
    import ctypes
    h = ctypes.c_void_p()
    st = api._lib.pspmm_pcsr_load(os.fsencode(str(p)), None, ctypes.byref(h))
    assert st == api.PSPMM_ERR_INVALID_ARG and not h.value
    assert "size" in api._lib.pspmm_last_error().decode()


def test_host_allocation_failure_returns_oom():
    """pspmm_reorder (host BFS) under an address-space limit too small for
    its O(n + nnz) work arrays: the entry returns PSPMM_ERR_OOM (status 8)
    and the process survives (an escaped std::bad_alloc would abort it)."""
    code = textwrap.dedent(f"""
        import resource, sys
        sys.path.insert(0, {ROOT!r})
        import numpy as np
        from paper_2605_15695_b200 import api
        n = 4_000_000
        rowptr = np.arange(n + 1, dtype=np.int32)            # a path: i -> i + 1
        colidx = np.minimum(np.arange(n, dtype=np.int32) + 1, n - 1)
        colidx[-1] = n - 2
        perm = np.empty(n, np.int32)
        vm = [int(l.split()[1]) for l in open('/proc/self/status') if l.startswith('VmSize')][0]
        resource.setrlimit(resource.RLIMIT_AS, ((vm << 10) + (24 << 20),) * 2)
        st = api._lib.pspmm_reorder(n, rowptr.ctypes.data_as(api._P),
                                    colidx.ctypes.data_as(api._P), 1, perm.ctypes.data_as(api._P))
        print("STATUS", st, api._lib.pspmm_last_error().decode())
    """)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.returncode, r.stderr[-2000:])
    m = re.search(r"STATUS (\d+) (.*)", r.stdout)
    assert m, r.stdout
    from paper_2605_15695_b200 import api
    assert int(m.group(1)) == api.PSPMM_ERR_OOM, r.stdout
    assert "reorder" in m.group(2)


def _definitions(src):
    return [m for m in re.finditer(r'^(?:extern "C" )?pspmm_status (pspmm_\w+)\([^;{]*\)\s*\{\n(.*)\n',
                                   src, re.M)]


def test_every_status_entry_is_guarded():
    found = set()
    for f in sorted(os.listdir(CSRC)):
        if not f.endswith((".cu", ".cpp")) or f.startswith("baseline_"):
            continue
        src = open(os.path.join(CSRC, f)).read()
        for m in _definitions(src):
            found.add(m.group(1))
            assert "pspmm::guarded(" in m.group(2), f"{f}: {m.group(1)} is not guarded"
    hdr = open(os.path.join(ROOT, "include", "pspmm.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    declared = set(re.findall(r"pspmm_status\s+(pspmm_\w+)\s*\(", hdr))
    assert declared and declared <= found, declared - found
