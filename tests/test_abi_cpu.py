"""Host-side checks that need no GPU: the C-ABI library loads, exports every
symbol include/impm_gpu.h declares, the struct layouts match the header, the
host utilities mirror the reference, and the product has no CPU fallback."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "impm_gpu.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(impm_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2507_09435_b200 import build

    build.build()
    from paper_2507_09435_b200 import _abi

    return _abi.lib()


def test_library_exports_every_header_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(REPO, "paper_2507_09435_b200",
                                                                        "libimpm_gpu.so")],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (impm_[a-z0-9_]+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing


def test_python_binding_covers_header(lib):
    from paper_2507_09435_b200 import _abi

    assert set(header_symbols()) <= set(_abi.EXPORTED) | {"impm_create_error"}


def test_struct_layouts_match_header(tmp_path):
    """ctypes structs vs the C compiler's view of include/impm_gpu.h."""
    from paper_2507_09435_b200 import _abi

    src = tmp_path / "layout.c"
    src.write_text("""
#include <stddef.h>
#include <stdio.h>
#include "impm_gpu.h"
#define P(T, f) printf(#T "." #f " %zu\\n", offsetof(T, f))
int main(void) {
  printf("impm_grid %zu\\nimpm_material %zu\\nimpm_options %zu\\nimpm_step_record %zu\\n",
         sizeof(impm_grid), sizeof(impm_material), sizeof(impm_options), sizeof(impm_step_record));
  P(impm_grid, origin); P(impm_grid, h); P(impm_material, E); P(impm_options, krylov_rtol);
  P(impm_options, profile); P(impm_step_record, rel_residuals); P(impm_step_record, nnz_assembled);
  return 0;
}""")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(REPO, "include"), "-o", str(exe), str(src)], check=True)
    got = dict(line.rsplit(" ", 1) for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                              check=True).stdout.split("\n") if line)
    got = {k: int(v) for k, v in got.items()}
    assert got["impm_grid"] == ctypes.sizeof(_abi.Grid)
    assert got["impm_material"] == ctypes.sizeof(_abi.Material)
    assert got["impm_options"] == ctypes.sizeof(_abi.Options)
    assert got["impm_step_record"] == ctypes.sizeof(_abi.StepRecordC)
    assert got["impm_grid.origin"] == _abi.Grid.origin.offset
    assert got["impm_grid.h"] == _abi.Grid.h.offset
    assert got["impm_material.E"] == _abi.Material.E.offset
    assert got["impm_options.krylov_rtol"] == _abi.Options.krylov_rtol.offset
    assert got["impm_options.profile"] == _abi.Options.profile.offset
    assert got["impm_step_record.rel_residuals"] == _abi.StepRecordC.rel_residuals.offset
    assert got["impm_step_record.nnz_assembled"] == _abi.StepRecordC.nnz_assembled.offset


def test_particle_layout_matches_reference_sizeof():
    from paper_2507_09435_b200 import particle_doubles

    # sizeof(impm::Particle<D>) = 232 / 304 / 392 bytes
    assert [particle_doubles(d) * 8 for d in (1, 2, 3)] == [232, 304, 392]


def test_version_and_sizes_callable_without_gpu(lib):
    assert b"sm_100a" in lib.impm_version()
    assert lib.impm_particle_doubles(3) == 49


def test_create_without_gpu_fails_loudly(lib):
    import paper_2507_09435_b200 as impm
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    grid = impm.GridSpec(2, (-1.0, -1.0), 1.0, (5, 5))
    parts = impm.seed_box(grid, (0.0, 0.0), (2.0, 2.0), 2, 1000.0)
    with pytest.raises(impm.CudaError):
        impm.MpmSim(grid, parts, impm.MaterialSpec("neo_hookean", impm.ElasticParams(1e6, 0.3)))


def test_missing_extension_raises(monkeypatch, tmp_path):
    from paper_2507_09435_b200 import _abi

    monkeypatch.setattr(_abi, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(_abi, "_lib", None)
    with pytest.raises(_abi.ExtensionMissing):
        _abi.lib()


def test_seed_box_matches_reference_fixture():
    import golden_util as gu
    import paper_2507_09435_b200 as impm

    fx = gu.load("cfg1_nh")
    dim, grid, mat, opts, parts, fixed, grav, spec = gu.problem(fx)
    g = impm.GridSpec(dim, grid["origin"], grid["h"], grid["nodes"])
    mine = impm.seed_box(g, (0.0, 0.0), (64.0, 64.0), 2, 2000.0)
    np.testing.assert_array_equal(mine, parts)


def test_gimp_weight_known_answers():
    import paper_2507_09435_b200 as impm

    w, dw = impm.gimp_weight_1d(0.0, 0.25, 1.0)  # tests/python/test_smoke.py:29-35
    assert abs(w - 0.875) < 1e-12 and dw == 0.0
    assert impm.block_size("gimp") == 5 and impm.block_size("linear") == 3
    assert impm.block_size("cubic-bspline") == 7
    with pytest.raises(impm.ConfigError):
        impm.gimp_weight_1d(0.0, 0.6, 1.0)


def build_facade_smoke(out_path):
    """Compiles tests/cpp/facade_smoke.cpp against include/impm_gpu.hpp and
    libimpm_gpu.so (the C++ drop-in facade)."""
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(REPO, "include"), "-o", out_path,
                    os.path.join(REPO, "tests", "cpp", "facade_smoke.cpp"),
                    "-L", os.path.join(REPO, "paper_2507_09435_b200"), "-limpm_gpu",
                    "-Wl,-rpath," + os.path.join(REPO, "paper_2507_09435_b200")], check=True)
    return out_path


def test_cpp_facade_compiles_and_links(lib, tmp_path):
    assert os.path.exists(build_facade_smoke(str(tmp_path / "facade_smoke")))


REF_INCLUDE = "/root/reference/proj/include"


@pytest.mark.skipif(not os.path.isdir(REF_INCLUDE), reason="reference headers not present (GPU box)")
def test_integration_snippet_compiles_against_reference(lib, tmp_path):
    """INTEGRATION.md section 1's snippet, verbatim, compiled in
    IMPM_GPU_REFERENCE_TYPES mode against the reference's own headers and
    linked with libimpm_gpu.so: impm_gpu::MpmSim<D> takes impm::Grid<D>,
    impm::Particle<D>, impm::MaterialSpec and impm::SolverOptions
    (mpm_solver.hpp:20-68)."""
    text = open(os.path.join(REPO, "INTEGRATION.md")).read()
    block = text.split("<!-- snippet:reference-types -->", 1)[1].split("<!-- /snippet -->", 1)[0]
    code = block.split("```cpp", 1)[1].split("```", 1)[0]
    src = tmp_path / "snippet.cpp"
    src.write_text(code + "\nint main() { return settle_column(0) == 12345.0; }\n")
    exe = tmp_path / "snippet"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(REPO, "include"), "-I", REF_INCLUDE,
                    "-o", str(exe), str(src), "-L", os.path.join(REPO, "paper_2507_09435_b200"), "-limpm_gpu"],
                   check=True)
    assert exe.exists()


@pytest.mark.skipif(not os.path.isdir(REF_INCLUDE), reason="reference headers not present (GPU box)")
def test_bar_swap_builds_against_reference(lib):
    """tests/cpp/bar_swap.cpp (the reference's build_bar/run_bar with only the
    MpmSim type swapped) builds against the reference headers; the binary
    travels to the GPU box for tests/test_gpu_facade.py."""
    from paper_2507_09435_b200 import build

    assert os.path.exists(build.build_bar_swap())
