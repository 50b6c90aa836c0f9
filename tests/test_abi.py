"""CPU-side checks of the drop-in boundary: libfpr_b200.so loads, exports every
symbol include/fpr_b200.h declares, and the ctypes struct layouts match the C
header (compiled with gcc here).  No compute calls -- no GPU needed."""
import ctypes as C
import os
import re
import subprocess

import pytest

import paper_2203_09284_b200 as fb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fpr_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(fpr_b200_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = fb.lib()
    names = declared_functions()
    assert len(names) >= 12
    for name in names:
        assert hasattr(L, name), name
    assert set(names) == set(fb.EXPORTS)


def test_struct_layouts_match_header(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(f"""
#include <stdio.h>
#include <stddef.h>
#include "{HEADER}"
int main(void) {{
  printf("%zu %zu %zu %zu %zu\\n", sizeof(fpr_graph_view), sizeof(fpr_config),
         sizeof(fpr_b200_options), sizeof(fpr_b200_result), sizeof(fpr_gen_params));
  printf("%zu %zu %zu\\n", offsetof(fpr_b200_options, stream), offsetof(fpr_b200_result, solve_ms),
         offsetof(fpr_gen_params, seed));
  printf("%zu %zu\\n", sizeof(fpr_parse_error), offsetof(fpr_parse_error, message));
  return 0;
}}
""")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-o", str(exe), str(src)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    sizes = [int(x) for x in out]
    assert sizes[:5] == [C.sizeof(fb._GraphView), C.sizeof(fb._Config), C.sizeof(fb._Options),
                         C.sizeof(fb._Result), C.sizeof(fb._GenParams)]
    assert sizes[5] == fb._Options.stream.offset
    assert sizes[6] == fb._Result.solve_ms.offset
    assert sizes[7] == fb._GenParams.seed.offset
    assert sizes[8:10] == [C.sizeof(fb._ParseErr), fb._ParseErr.message.offset]


def test_library_is_sm100a_only():
    """The fatbin carries sm_100a SASS (no PTX JIT fallback, no other arch)."""
    out = subprocess.run(["cuobjdump", "--list-elf", fb.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_\d+a?", out.stdout))
    assert arches == {"sm_100a"}, arches


def test_engine_tags_roundtrip():
    for k in fb.EngineKind:
        assert fb.parse_engine(fb.to_string(k)) is k
    with pytest.raises(ValueError, match="unknown engine tag"):
        fb.parse_engine("gpu")


def test_cpu_engine_rejected_without_device_work():
    g = fb.Graph(1, 0, __import__("numpy").array([0, 0], "u8"), __import__("numpy").zeros(0, "u8"),
                 __import__("numpy").array([0], "u8"))
    with pytest.raises(ValueError, match="reference CPU engine"):
        fb.run_engine("ec_seq", g, fb.PageRankConfig())


def test_metrics_mirror():
    import numpy as np

    assert fb.l1_norm([1.0, 2.0], [1.5, 1.0]) == 1.5
    assert fb.linf_norm([1.0, 2.0], [1.5, 1.0]) == 1.0
    with pytest.raises(ValueError, match="length mismatch"):
        fb.l1_norm(np.zeros(2), np.zeros(3))


def test_every_pointer_entry_point_has_argtypes():
    """ctypes passes an un-declared Python int as a 32-bit C int, silently
    truncating device pointers; lib() must declare every entry point that
    takes arguments (a part created without the partition path once hit it)."""
    L = fb.lib()
    no_args = {"fpr_b200_last_error", "fpr_b200_version"}
    for name in fb.EXPORTS:
        if name in no_args:
            continue
        assert getattr(L, name).argtypes is not None, name


def test_option_flags_match_header():
    """The Python flag constants are the header's, and `reorder` maps to the
    two reorder flags (anything else is rejected before any device work)."""
    text = open(HEADER).read()
    for name, val in (("REORDER", fb.OPT_REORDER), ("PULL", fb.OPT_PULL), ("PB", fb.OPT_PB),
                      ("REORDER_SOURCES", fb.OPT_REORDER_SOURCES)):
        m = re.search(rf"#define FPR_B200_OPT_{name} (\d+)u", text)
        assert m and int(m.group(1)) == val, name
    assert fb._options(reorder=True).flags == fb.OPT_REORDER
    assert fb._options(reorder="degree").flags == fb.OPT_REORDER
    assert fb._options(reorder="sources", pb=True).flags == fb.OPT_REORDER_SOURCES | fb.OPT_PB
    assert fb._options().flags == 0  # the library picks the sweep kind
    assert fb._options(pb=False).flags == fb.OPT_PULL
    for name, val in (("PULL", fb.SWEEP_PULL), ("PB", fb.SWEEP_PB)):
        m = re.search(rf"#define FPR_B200_SWEEP_{name} (\d+)", text)
        assert m and int(m.group(1)) == val, name
    with pytest.raises(ValueError, match="reorder"):
        fb._options(reorder="bfs")
