"""C-ABI boundary checks that need no GPU: the library loads and exports every symbol
declared in include/gc.h, and the binding's structs match the header's field lists."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "gc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gc_[a-z_]+)\s*\(", src)))


def test_header_declares_boundary():
    fns = header_functions()
    for f in ("gc_create", "gc_destroy", "gc_solve_batch", "gc_solve_batch_host", "gc_last_error"):
        assert f in fns


def test_library_exports_every_symbol():
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_1008_0502_b200", "libgc.so"))
    for f in header_functions():
        assert hasattr(lib, f), f


def test_binding_names_match_header():
    import paper_1008_0502_b200 as gc
    for f in header_functions():
        assert hasattr(gc, f), f
    assert set(gc.EXPORTED) == set(header_functions())


def test_struct_layout_matches_header():
    import paper_1008_0502_b200 as gc
    src = open(os.path.join(ROOT, "include", "gc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    body = re.search(r"typedef struct \{([^{}]*)\} gc_batch;", src, re.S).group(1)
    names = re.findall(r"\*?\s*([a-z_A-Z]+)\s*[,;]", body)
    assert [n for n, _ in gc.gc_batch._fields_] == names
    body = re.search(r"typedef struct \{([^{}]*)\} gc_seq_batch;", src, re.S).group(1)
    names = re.findall(r"\*?\s*([a-z_A-Z]+)\s*[,;]", body)
    assert [n for n, _ in gc.gc_seq_batch._fields_] == names
    body = re.search(r"typedef struct \{([^{}]*)\} gc_energy_batch;", src, re.S).group(1)
    names = re.findall(r"\*?\s*([a-z_A-Z]+)\s*[,;]", body)
    assert [n for n, _ in gc.gc_energy_batch._fields_] == names
    import ctypes
    assert ctypes.sizeof(gc.gc_gmm) == 8 + 8 * 4 + 24 * 4 + 48 * 4
    body = re.search(r"typedef struct \{([^{}]*)\} gc_saliency_batch;", src, re.S).group(1)
    names = re.findall(r"\*?\s*([a-z_A-Z0-9]+)\s*[,;]", body)
    assert [n for n, _ in gc.gc_saliency_batch._fields_] == names
    body = re.search(r"typedef struct \{([^{}]*)\} gc_prior_params;", src, re.S).group(1)
    names = re.findall(r"int\s+([a-z_A-Z]+)", body)
    assert [n for n, _ in gc.gc_prior_params._fields_] == names
    body = re.search(r"typedef struct \{([^{}]*)\} gc_config;", src, re.S).group(1)
    names = re.findall(r"([a-z_]+)\s*[,;]", body)
    assert [n for n, _ in gc.gc_config._fields_] == names


def test_library_is_sm100a():
    """The shared object embeds sm_100a SASS (cuobjdump lists it) -- no PTX-only JIT path."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        return
    out = subprocess.run([exe, "--list-elf", os.path.join(ROOT, "paper_1008_0502_b200", "libgc.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_oracle_not_imported_by_product():
    """The product path must never route through the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_1008_0502_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle.cpp" not in txt, f


def test_binding_constants_match_header():
    """The binding's copies of the header's limits (no GPU needed)."""
    import paper_1008_0502_b200 as gc
    src = open(os.path.join(ROOT, "include", "gc.h")).read()
    defs = dict(re.findall(r"#define (GC_[A-Z_]+) (.+)", src))
    assert gc.PARTS_MAX == int(defs["GC_PARTS_MAX"])
    assert gc.GMM_MAX == int(defs["GC_GMM_MAX"])
    assert gc.PRIOR_RMAX == int(defs["GC_PRIOR_RMAX"])
    assert defs["GC_CAP_MAX"].strip() == "((1 << 26) - 1)" and gc.CAP_MAX == (1 << 26) - 1
