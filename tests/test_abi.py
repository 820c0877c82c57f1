"""The C-ABI library loads without a GPU and exports every function pg.h declares."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "pg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pg_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_1404_1521_b200 import build
    return build.build()


def test_header_declares_north_star_entry_points():
    names = declared()
    for n in ("pg_init", "pg_train_step", "pg_score"):
        assert n in names


def test_every_declared_symbol_exported(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (pg_\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing


def test_binding_loads_and_names_match(libpath):
    import paper_1404_1521_b200 as pg
    L = pg.lib()
    assert L.pg_abi_version() == 1
    assert sorted(pg.EXPORTED) == declared()
    for n in declared():
        assert callable(getattr(pg, n)), n


def test_no_gpu_compute_fails_loudly(libpath):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1404_1521_b200 as pg
    with pytest.raises(pg.PGError):
        pg.pg_init(100, 8, 5, 4, 1)


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1404_1521_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).lower() or f == "__init__.py" and \
                    "import oracle" not in txt, f


def test_header_constants_match_binding():
    """Every PG_* enumerator in pg.h has the same value in the Python binding."""
    import paper_1404_1521_b200 as pg
    src = open(os.path.join(ROOT, "include", "pg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    consts = {}
    for body in re.findall(r"enum\s*\w*\s*\{(.*?)\}", src, flags=re.S):
        nxt = 0
        for item in [x.strip() for x in body.split(",") if x.strip()]:
            m = re.match(r"(PG_\w+)\s*(?:=\s*(-?\d+))?$", item)
            assert m, item
            val = int(m.group(2)) if m.group(2) is not None else nxt
            consts[m.group(1)] = val
            nxt = val + 1
    for name in ("PG_OK", "PG_ERANGE", "PG_EDIVERGED", "PG_SCATTER_DET", "PG_SCATTER_ATOMIC", "PG_OPT_SCATTER",
                 "PG_OPT_RESERVE", "PG_OPT_ACTIVATION", "PG_OPT_REDUCTION", "PG_ACT_HARDTANH", "PG_ACT_TANH",
                 "PG_REDUCE_MEAN", "PG_REDUCE_SUM"):
        assert name in consts, name
    for name, val in consts.items():
        if hasattr(pg, name):
            assert getattr(pg, name) == val, (name, getattr(pg, name), val)
