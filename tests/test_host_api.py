"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/acs_gpu.h declares; the TSPLIB parser behind it matches the
reference parser (coordinates, field-naming ParseError messages); the C++
drop-in API compiles against the reference include path and round-trips
instances; without a GPU every compute entry point fails loudly (no CPU
fallback)."""
import os
import re
import subprocess

import numpy as np
import pytest

import oracle as O
from helpers import TSPLIB

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(REPO, "include", "acs_gpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(acs_[a-z0-9_]+)\s*\(", text)))


def test_every_header_symbol_is_exported(acs):
    names = header_functions()
    assert len(names) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", acs.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, f"not exported: {missing}"
    from paper_1605_02669_b200 import _native as N
    assert set(N.SIGNATURES) == set(names)
    assert acs.lib().acs_gpu_abi_version() == 5


def test_library_is_sm100a(acs):
    out = subprocess.run(["cuobjdump", "--list-elf", acs.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("name", TSPLIB)
def test_parse_matches_reference_loader(acs, name):
    text = O.read_tsplib_text(name)
    inst = acs.parse_tsplib(text)
    I = O.parse_coords(text)
    assert inst.name == name and inst.n == I.n and inst.edge_weight_type == I.type
    assert np.array_equal(inst.xs, I.xs) and np.array_equal(inst.ys, I.ys)
    if O.Reference.available():
        ri, err = O.Reference().parse(text)
        xs, ys = ri.coords()
        assert err is None and np.array_equal(xs, inst.xs) and np.array_equal(ys, inst.ys)


BAD = [
    "NAME: x\nEDGE_WEIGHT_TYPE: EUC_2D\nNODE_COORD_SECTION\n1 0 0\nEOF\n",
    "NAME: x\nDIMENSION: 3\nNODE_COORD_SECTION\n1 0 0\n",
    "NAME: x\nDIMENSION: 3\nEDGE_WEIGHT_TYPE: GEO\n",
    "NAME: x\nDIMENSION: abc\n",
    "NAME: x\nDIMENSION: 0\n",
    "DIMENSION: 3\nEDGE_WEIGHT_TYPE: EUC_2D\nNODE_COORD_SECTION\n1 0 0\n2 1 1\nEOF\n",
    "DIMENSION: 2\nEDGE_WEIGHT_TYPE: EUC_2D\nNODE_COORD_SECTION\n1 0 0\n2 1 1\n3 2 2\n",
    "DIMENSION: 3\nEDGE_WEIGHT_TYPE: EUC_2D\nNODE_COORD_SECTION\n1 0 0\n2 one 1\n3 2 2\n",
    "DIMENSION: 2\nEDGE_WEIGHT_TYPE: EUC_2D\nNODE_COORD_SECTION\n1 0 0\n2 1 1\nEOF\n",
    "EDGE_WEIGHT_TYPE: EUC_2D\n",
    "DIMENSION : 3\nEDGE_WEIGHT_TYPE : ATT\n",
]


@pytest.mark.parametrize("text", BAD)
def test_parse_errors_match_reference(acs, ref, text):
    _, want = ref.parse(text)
    assert want is not None
    with pytest.raises(acs.ParseError) as e:
        acs.parse_tsplib(text)
    assert str(e.value) == want


GOOD_FORMS = [
    "NAME: t\nDIMENSION: 3\nEDGE_WEIGHT_TYPE: EUC_2D\nNODE_COORD_SECTION\n1 0 0\n2 3 4\n3 0 8\nEOF\n",
    "NAME : t\nTYPE : TSP\nCOMMENT : a: b\nDIMENSION : 3\nEDGE_WEIGHT_TYPE : CEIL_2D\nNODE_COORD_SECTION\n"
    "1 0.5 0\n  2 3 4.25  \n\n3 0 8\n",
    "NAME t\nDIMENSION 4\nEDGE_WEIGHT_TYPE ATT\nNODE_COORD_SECTION\n1 1e3 2\n2 3 4\n3 0 8\n4 -7 2.5\nEOF\nGARBAGE\n",
]


@pytest.mark.parametrize("text", GOOD_FORMS)
def test_parse_header_forms(acs, text):
    inst = acs.parse_tsplib(text)
    if O.Reference.available():
        ri, err = O.Reference().parse(text)
        assert err is None and ri.name == inst.name and ri.type == inst.edge_weight_type
        xs, ys = ri.coords()
        assert np.array_equal(xs, inst.xs) and np.array_equal(ys, inst.ys)


def test_no_cpu_fallback_without_gpu(acs):
    if acs.device_count() > 0:
        pytest.skip("a GPU is visible")
    inst = acs.parse_tsplib(GOOD_FORMS[0])
    with pytest.raises(acs.AcsError) as e:
        acs.build_candidates(inst, 32)
    assert e.value.code == -2
    with pytest.raises(acs.AcsError):
        acs.Colony(inst, acs.AcsParams())


def test_invalid_params_rejected(acs):
    inst = acs.parse_tsplib(GOOD_FORMS[0])
    for bad in (dict(cl=0), dict(cl=33), dict(k=0), dict(rho=0.0), dict(alpha=1.0), dict(q0=1.5),
                dict(variant="spm", s=3)):
        with pytest.raises(acs.AcsError) as e:
            acs.Colony(inst, acs.AcsParams(**bad))
        assert e.value.code == -1, bad


CPP_TEST = r"""
#include <cassert>
#include <cstdio>
#include <sstream>
#include "acs/tsp_instance.hpp"
#include "acs/rng.hpp"
#include "acs/solver.hpp"
int main(int argc, char **argv) {
    acs::TspInstance a = acs::load_tsplib_file(argv[1]);
    acs::TspInstance b = acs::parse_tsplib(acs::serialize_tsplib(a));
    assert(a.xs_ == b.xs_ && a.ys_ == b.ys_ && a.dimension_ == b.dimension_ && a.name_ == b.name_);
    std::vector<uint32_t> id(a.dimension_);
    for (uint32_t i = 0; i < a.dimension_; ++i) id[i] = i;
    std::printf("%lld %d %s\n", (long long)a.tour_length(id), a.distance(0, 1), acs::to_string(a.edge_weight_type_));
    acs::RngStream r = acs::RngStream::derive(42, 1, 7);
    unsigned long long x = r.next_u64();
    std::printf("%016llx %llu\n", x, (unsigned long long)r.uniform_int(280));
    std::istringstream cat("# c\nd198 15780\npr2392 378032 # x\nbad\n");
    auto m = acs::load_optimum_catalog(cat);
    std::printf("%zu %lld %.6f %d\n", m.size(), (long long)m["pr2392"], acs::default_q0(1379),
                (int)acs::select_best(std::vector<int64_t>{10, 7, 9}));
    try { acs::parse_tsplib(std::string("DIMENSION: 3\n")); } catch (const acs::ParseError &e) { std::printf("%s\n", e.what()); }
    return 0;
}
"""


def test_cpp_dropin_api(acs, tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text(CPP_TEST)
    exe = tmp_path / "t"
    lib_dir = os.path.dirname(acs.LIB_PATH)
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O1", f"-I{REPO}/include", str(src), "-o", str(exe),
                    f"-L{lib_dir}", "-lacs_b200", f"-Wl,-rpath,{lib_dir}"], check=True)
    path = os.path.join(REPO, "data", "tsplib", "pr2392.tsp.gz")
    out = subprocess.run([str(exe), path], capture_output=True, text=True, check=True).stdout.split("\n")
    I = O.load("pr2392")
    assert out[0] == f"378032 {O.Oracle().distance(I, 0, 1)} EUC_2D"
    assert out[1] == "1e41e6edf5d70818 133"
    assert out[2] == "2 378032 0.985497 1"
    assert out[3] == "EDGE_WEIGHT_TYPE: missing"


def test_serialize_matches_reference(acs, ref, tmp_path):
    """byte-identical TSPLIB text from the C++ drop-in serialize_tsplib"""
    src = tmp_path / "s.cpp"
    src.write_text('#include <cstdio>\n#include "acs/tsp_instance.hpp"\nint main(int, char **v) {'
                   ' std::fputs(acs::serialize_tsplib(acs::load_tsplib_file(v[1])).c_str(), stdout); }\n')
    lib_dir = os.path.dirname(acs.LIB_PATH)
    subprocess.run(["/usr/bin/g++", "-std=c++20", f"-I{REPO}/include", str(src), "-o", str(tmp_path / "s"),
                    f"-L{lib_dir}", "-lacs_b200", f"-Wl,-rpath,{lib_dir}"], check=True)
    for name in ("d198", "att532", "pr2392"):
        out = subprocess.run([str(tmp_path / "s"), os.path.join(REPO, "data", "tsplib", f"{name}.tsp.gz")],
                             capture_output=True, text=True, check=True).stdout
        ri, _ = ref.parse(O.read_tsplib_text(name))
        assert out == ri.serialize()


def test_random_instance_matches_reference_stream(acs):
    """rnd10k from the product generator equals the
    oracle's draw sequence; first node pinned by the reference probe (App. A)."""
    a = acs.random_uniform_instance(10000)
    b = O.rnd_instance(10000)
    assert a.name == "rnd10k" and (a.xs[0], a.ys[0]) == (120054.0, 324231.0)
    assert np.array_equal(a.xs, b.xs) and np.array_equal(a.ys, b.ys)
    assert acs.load_instance("rnd10k").n == 10000


def test_product_loaders(acs):
    cat = acs.optima()
    assert cat["pr2392"] == 378032 and cat["d198"] == 15780
    inst = acs.load_instance("pr2392")
    I = O.load("pr2392")
    assert inst.n == 2392 and inst.optimum == 378032
    assert np.array_equal(inst.xs, I.xs) and np.array_equal(inst.ys, I.ys)


def test_bench_product_path_does_not_use_the_oracle():
    """Only the cpu_baseline leg and the --impl reference arm may touch oracle/."""
    import ast
    tree = ast.parse(open(os.path.join(REPO, "bench.py")).read())
    allowed = {"cpu_baseline_seq", "run_reference"}
    for fn in ast.walk(tree):
        if isinstance(fn, ast.FunctionDef) and fn.name not in allowed:
            for node in ast.walk(fn):
                if isinstance(node, (ast.Import, ast.ImportFrom)):
                    mods = [a.name for a in node.names] if isinstance(node, ast.Import) else [node.module or ""]
                    assert not any(m.split(".")[0] == "oracle" for m in mods), fn.name


CPP_STATS = r"""
#include <cstdio>
#include <vector>
#include "acs/stats.hpp"
#include "acs/solver.hpp"
#include "acs/tsp_instance.hpp"
int main() {
    const std::vector<double> a{1, 2, 3}, b{4, 5, 6};
    std::printf("%.6f %.6f\n", acs::rank_sum_test(a, b), acs::mann_whitney_u(a, b));
    const std::vector<int64_t> len{2579, 2600, 2650};
    const acs::SampleSummary s = acs::summarize(len, 2579);
    std::printf("%.4f %.4f %lld %u\n", s.mean_error_pct, s.min_error_pct, (long long)s.best_length, s.runs);
    const std::vector<double> good{1, 1.5, 2, 2.5, 3, 1.2, 1.1}, bad{5, 6, 7, 8, 9, 5.5, 6.5};
    std::printf("%c%c\n", acs::significance_mark(good, bad), acs::significance_mark(bad, good));
    const acs::TspInstance r = acs::random_uniform_instance(10000);
    std::printf("%s %.0f %.0f %.2f\n", r.name_.c_str(), r.xs_[0], r.ys_[0], acs::relative_error(102, 100));
    const auto cat = acs::load_optimum_catalog_file(ACS_CATALOG);
    std::printf("%lld\n", (long long)cat.at("pr2392"));
    return 0;
}
"""


def test_cpp_stats_and_generators(acs, tmp_path):
    src = tmp_path / "st.cpp"
    src.write_text(CPP_STATS)
    lib_dir = os.path.dirname(acs.LIB_PATH)
    cat = os.path.join(REPO, "data", "tsplib", "optima.txt.gz")
    subprocess.run(["/usr/bin/g++", "-std=c++20", f"-I{REPO}/include", f'-DACS_CATALOG="{cat}"', str(src),
                    "-o", str(tmp_path / "st"), f"-L{lib_dir}", "-lacs_b200", f"-Wl,-rpath,{lib_dir}"], check=True)
    out = subprocess.run([str(tmp_path / "st")], capture_output=True, text=True, check=True).stdout.split("\n")
    assert out[0] == "0.100000 0.000000"
    assert out[1] == f"{100 * (2609.6666666666665 - 2579) / 2579:.4f} 0.0000 2579 3"
    assert out[2] == "+-"
    assert out[3] == "rnd10k 120054 324231 2.00"
    assert out[4] == "378032"
