"""Host-side check (no GPU): the ctypes mirrors of the C ABI structs in the Python binding have the
fields of include/flexctc.h in the same order with the same C types, so a config field added on one
side only (as merge_first was, round 2) cannot silently shift the others."""
import ctypes
import os
import re

from tests.conftest import ROOT

CT = {"int32_t": ctypes.c_int32, "float": ctypes.c_float, "int64_t": ctypes.c_int64, "double": ctypes.c_double}


def _c_struct(name):
    src = open(os.path.join(ROOT, "include", "flexctc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)  # drop comments
    m = re.search(r"typedef struct \{([^}]*)\}\s*" + name + ";", src)
    assert m, name
    fields = []
    for decl in m.group(1).split(";"):
        decl = decl.strip()
        if not decl:
            continue
        typ, rest = decl.split(None, 1)
        for f in rest.split(","):
            fields.append((f.strip(), CT[typ]))
    return fields


def test_config_layout_matches_header():
    from paper_2508_07315_b200 import flexctc
    assert [(n, t) for n, t in flexctc.Config._fields_] == _c_struct("flexctc_config")


def test_lm_info_layout_matches_header():
    from paper_2508_07315_b200 import flexctc
    assert [(n, t) for n, t in flexctc.LmInfo._fields_] == _c_struct("flexctc_lm_info")


def test_oracle_cfg_layout_matches_header():
    import oracle
    src = open(os.path.join(ROOT, "oracle", "oracle.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    m = re.search(r"typedef struct \{([^}]*)\}\s*oracle_cfg;", src)
    fields = [(d.split()[1], CT[d.split()[0]]) for d in (x.strip() for x in m.group(1).split(";")) if d]
    assert [(n, t) for n, t in oracle.Cfg._fields_] == fields
