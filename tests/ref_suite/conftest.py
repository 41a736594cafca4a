"""The reference's own hot-path tests, run UNCHANGED against the drop-in.

The files next to this conftest are byte-identical copies of
``/root/reference/pkg/tests/test_{aosoa,binning,neighbors,decomp,md,
acceptance,cli}.py`` (VERDICT r1 "next" #8).  They
import ``particula``; this conftest binds that name and its submodules to
``paper_2109_09056_b200`` before collection, so every call goes through the
C ABI into the sm_100a kernels (there is no CPU fallback: the tests need a
GPU and are marked ``gpu``).

Tests of subsystems outside the north-star path (grid/P2G, pencil
FFT, SPME mesh, PIC and their CLI runners) are skipped with that reason; the
modules they import are bound to empty placeholders so the files import
unchanged.  Every other test must pass.
"""

import sys
import types

import pytest

import paper_2109_09056_b200 as _pkg
from paper_2109_09056_b200 import cli as _cli

_OUT_OF_SCOPE = ("grid", "pfft", "pic")


def _bind():
    root = types.ModuleType("particula")
    root.__path__ = []
    root.__doc__ = "particula -> paper_2109_09056_b200 (tests/ref_suite/conftest.py)"
    subs = {name: getattr(_pkg, name) for name in _pkg.__all__}
    subs["cli"] = _cli
    for name in _OUT_OF_SCOPE:
        m = types.ModuleType(f"particula.{name}")
        m.__doc__ = "out of scope for the MD hot path (SURVEY §2)"
        subs[name] = m
    for name, mod in subs.items():
        setattr(root, name, mod)
        sys.modules[f"particula.{name}"] = mod
    sys.modules["particula"] = root


_bind()

# test -> reason (out-of-scope subsystems only)
SKIP = {
    "test_criterion_02_layout_transparency":
        "its second half drives the CLI 'pic' runner (PIC: out of scope); the md half "
        "(V in {1,4,8,16,SoA}, bitwise rows) is tests/test_cli.py::test_layout_transparency",
    "test_criterion_05_spme_vs_direct_ewald": "SPME mesh (longrange.spme): out of scope",
    "test_criterion_06_distributed_fft": "pencil FFT (pfft): out of scope",
    "test_criterion_07_boris_pusher": "PIC (pic): out of scope",
    "test_criterion_08_implicit_energy_conservation": "PIC (pic): out of scope",
    "test_criterion_09_sgct_noise_reduction": "PIC sparse grids (pic): out of scope",
    "test_criterion_10_interpolation_suite": "grid P2G/G2P (grid): out of scope",
    "test_pic_implicit_csv_columns": "CLI pic-implicit runner: out of scope",
    "test_solver_failure_exit_4": "CLI pic-implicit solver failure: out of scope",
    "test_fft_bench_table": "CLI fft-bench runner: out of scope",
    "test_sgct_subcommand": "CLI sgct runner: out of scope",
    "test_spme_check_subcommand": "CLI spme-check runner: out of scope",
}


@pytest.hookimpl(tryfirst=True)
def pytest_collection_modifyitems(config, items):
    for item in items:
        if "ref_suite" not in str(item.fspath):
            continue
        item.add_marker(pytest.mark.gpu)
        base = item.name.split("[", 1)[0]
        if base in SKIP:
            item.add_marker(pytest.mark.skip(reason=SKIP[base]))
