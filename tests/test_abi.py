"""CPU checks of the drop-in boundary: the shared library loads without a GPU
and exports exactly the entry points include/chimera_b200.h declares, and the
ctypes structs match the C layouts."""

import ctypes
import os
import re

import pytest

from paper_2603_22206_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "chimera_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(chm_\w+)\s*\(", src, flags=re.M)))


def test_header_matches_binding_table():
    assert declared_functions() == sorted(_lib.EXPORTED_SYMBOLS)


def test_library_exports_every_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert _lib.load().chm_version().startswith(b"chimera_b200")
    assert _lib.load().chm_status_string(4) == b"duplicate request"


def _c_struct_fields(name):
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    m = re.search(r"typedef struct %s \{(.*?)\} %s;" % (name, name), src, flags=re.S)
    body = m.group(1)
    fields = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        decl = re.sub(r"\[[^\]]*\]", "", decl)
        for part in decl.split(","):
            fields.append(re.findall(r"(\w+)\s*$", part.strip())[0])
    return fields


@pytest.mark.parametrize("cname,pyt", [
    ("chm_pool", _lib.Pool), ("chm_balancer_cfg", _lib.BalancerCfg),
    ("chm_aging_cfg", _lib.AgingCfg), ("chm_monitor_state", _lib.MonitorState),
    ("chm_rows", _lib.Rows), ("chm_row_scratch", _lib.RowScratch),
    ("chm_decisions", _lib.Decisions), ("chm_queue_state", _lib.QueueState),
    ("chm_encoder_cfg", _lib.EncoderCfg), ("chm_encoder_weights", _lib.EncoderWeights),
    ("chm_encoder_workspace", _lib.EncoderWorkspace)])
def test_struct_field_order(cname, pyt):
    assert _c_struct_fields(cname) == [f[0] for f in pyt._fields_]
