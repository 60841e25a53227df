"""Host-side checks of the C-ABI library (no GPU needed): it loads and exports every entry
point declared in include/thermo.h; the binding fails loudly without a device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "thermo.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(thermo_[A-Za-z_]+)\s*\(", src)))


def test_header_declares_the_four_entry_points():
    names = _declared()
    for n in ("thermo_create_mesh", "thermo_set_bc", "thermo_step", "thermo_get_T"):
        assert n in names


def test_library_exports_every_declared_symbol():
    import __graft_entry__ as g
    g.build()
    from paper_1707_03581_b200 import thermo as T
    lib = ctypes.CDLL(T.LIB_PATH)
    for n in _declared():
        assert hasattr(lib, n), n
    assert sorted(T.EXPORTS) == _declared()


def test_oracle_is_not_imported_by_the_product_path():
    pkg = os.path.join(ROOT, "paper_1707_03581_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                bad = re.findall(r"^\s*(?:import oracle|from oracle\b|#\s*include\s*[<\"].*oracle)", txt, flags=re.M)
                assert not bad, (f, bad)


def test_create_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1707_03581_b200 import inputs as I
    from paper_1707_03581_b200.thermo import Thermo, ThermoError
    cfg = I.make_config("cfg0")
    with pytest.raises(ThermoError):
        Thermo.from_config(cfg, stream=0)
