"""CPU-only checks of the drop-in boundary: the C-ABI library loads and exports
every symbol include/tinfer_sm100.h declares (no compute calls), and the ctypes
structures match the header's field order."""

import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "tinfer_sm100.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tf_[a-z_0-9]+)\s*\(", text)))


def header_struct_fields(name):
    text = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    body = re.search(r"typedef struct %s \{(.*?)\} %s;" % (name, name), text, flags=re.S).group(1)
    fields = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        # "int a, b" / "const void* x" / "size_t n"
        parts = decl.replace("*", " ").split()
        names = " ".join(parts[1:]).split(",") if "," in decl else [parts[-1]]
        if "," in decl:
            first = decl.split(",")[0].replace("*", " ").split()[-1]
            rest = [p.strip().replace("*", "") for p in decl.split(",")[1:]]
            names = [first] + rest
        fields += [n.strip() for n in names]
    return fields


def test_library_exports_every_declared_symbol():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2407_04991_b200 import _native as N
    lib = N.load_library()
    declared = header_functions()
    assert declared, "no tf_* functions parsed from the header"
    for name in declared:
        assert hasattr(lib, name), f"{name} not exported"
        assert name in N.SIGNATURES, f"{name} has no ctypes signature"
    assert set(N.SIGNATURES) == set(declared)
    assert lib.tf_abi_version() == N.ABI_VERSION


@pytest.mark.parametrize("cname,pyname", [("tf_gemm_desc", "GemmDesc"), ("tf_embed_desc", "EmbedDesc"),
                                          ("tf_layer_weights", "LayerWeights"),
                                          ("tf_model_desc", "ModelDesc"),
                                          ("tf_session_desc", "SessionDesc"),
                                          ("tf_beam_desc", "BeamDesc")])
def test_ctypes_structs_mirror_header(cname, pyname):
    from paper_2407_04991_b200 import _native as N
    py = [f[0] for f in getattr(N, pyname)._fields_]
    assert py == header_struct_fields(cname)


def test_sm100a_code_in_library():
    import subprocess
    from paper_2407_04991_b200 import _native as N
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", N.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for mnemonic in ("UTCHMMA", "UTMALDG", "LDTM"):  # tcgen05.mma, TMA, tcgen05.ld
        assert mnemonic in out, mnemonic
