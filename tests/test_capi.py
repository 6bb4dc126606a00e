"""CPU checks of the C-ABI boundary: the in-tree sm_100a library loads and
exports every function declared in include/duchess_b200.h, and the ctypes
struct layouts match the header's field lists."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "duchess_b200.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(duchess_\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    from paper_2509_24957_b200 import _lib
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.SYMBOLS, f"{name} missing from the ctypes binding"
    assert lib.duchess_version().decode().startswith("duchess_b200")


def _struct_fields(name):
    text = HEADER.read_text()
    body = re.search(r"typedef struct %s \{(.*?)\} %s;" % (name, name), text, flags=re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body)
    return re.findall(r"\b(\w+)\s*(?:\[\d+\])?\s*;", body)


@pytest.mark.parametrize("cname,pyname", [("DuchessPolicy", "Policy"),
                                          ("DuchessWorkload", "Workload"),
                                          ("DuchessState", "State")])
def test_struct_layouts_match_header(cname, pyname):
    from paper_2509_24957_b200 import _lib
    py = getattr(_lib, pyname)
    assert [f[0] for f in py._fields_] == _struct_fields(cname)


def test_workspace_queries_need_no_gpu():
    from paper_2509_24957_b200 import _lib
    lib = _lib.load()
    assert lib.duchess_score_workspace_bytes(4096, 1) == 0
    assert lib.duchess_score_workspace_bytes(4096, 2) == 4096 * 2 * 16 + 4096 * 4
    assert lib.duchess_fork_workspace_bytes(4, 8) == (3 * 4 + 32 + 4) * 4


def test_invalid_arguments_are_rejected_before_launch():
    from paper_2509_24957_b200 import _lib
    lib = _lib.load()
    # null pointers / bad sizes return DUCHESS_EINVAL (1) without touching a device
    assert lib.duchess_score(None, 1, 4, 1, 1, 16, 16, 16, 16, None, None, None, None, None,
                             None, 0, 0, 0, None) == 1
    assert lib.duchess_sort_difficulty(None, None, 1, None, None) == 1
    assert lib.duchess_lr_grad(None, 1, None, None, 8, 16, 1.0, None, None, 0, None) == 1
    assert lib.duchess_branch_out_sample(None, 0, 1.0, None, 0, None, None, None, None) == 1
    pol = _lib.Policy()
    pol.max_branches = 0
    assert lib.duchess_advance(ctypes.byref(pol), ctypes.byref(_lib.Workload()),
                               ctypes.byref(_lib.State()), None) == 1
    # round-2 entry points: unknown scorer flags, bad sort / KV / measurement arguments
    fake = ctypes.c_void_p(16)                   # never dereferenced: rejected first
    assert lib.duchess_score_active_ex(fake, 1, 4, 1, 1, 16, 16, 16, 16, fake, fake, fake,
                                       fake, fake, fake, 4, None) == 1
    assert lib.duchess_sort_keys(None, 5, None, None, 0, None) == 1
    assert lib.duchess_sort_keys(fake, 5, fake, fake, 8, None) == 1      # workspace too small
    assert lib.duchess_sort_keys(None, 0, None, None, 0, None) == 0       # empty: nothing to do
    assert lib.duchess_sort_keys_workspace_bytes(5) >= 5 * 24
    assert lib.duchess_kv_round(ctypes.byref(pol), ctypes.byref(_lib.State()),
                                ctypes.byref(_lib.KV()), None) == 1
    assert lib.duchess_gate(None, 1000, None, None) == 1
    assert lib.duchess_write_stream(None, 1 << 20, 0, None) == 1
    assert lib.duchess_row_normalize(fake, 7, 4, 16, fake, None) == 1     # unknown dtype
    rows = (ctypes.c_int32 * 3)(5, 1, 9)
    assert lib.duchess_upload_rows(None, fake, 64, rows, 3, 10, None) == 1
    assert lib.duchess_upload_rows(fake, fake, 64, rows, 3, 9, None) == 1    # row 9 out of range
    assert lib.duchess_upload_rows(fake, fake, 64, None, 0, 9, None) == 0    # nothing to copy


@pytest.mark.parametrize("cname,pyname", [("DuchessPolicy", "Policy"),
                                          ("DuchessWorkload", "Workload"),
                                          ("DuchessState", "State")])
def test_struct_offsets_match_c_compiler(cname, pyname, tmp_path):
    """Field offsets and sizes of the ctypes mirrors == what a C compiler lays out."""
    import shutil
    import subprocess
    from paper_2509_24957_b200 import _lib
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    py = getattr(_lib, pyname)
    fields = [f[0] for f in py._fields_]
    src = tmp_path / "off.c"
    src.write_text("#include <stdio.h>\n#include <stddef.h>\n#include \"duchess_b200.h\"\n"
                   "int main(void){\n" + "".join(
                       f'printf("%zu\\n", offsetof({cname}, {f}));\n' for f in fields)
                   + f'printf("%zu\\n", sizeof({cname}));return 0;}}\n')
    exe = tmp_path / "off"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [getattr(py, f).offset for f in fields] + [ctypes.sizeof(py)]
    assert got == want
