"""CPU-side checks of the boundary: libecho.so builds for sm_100a, loads, exports every symbol include/echo.h
declares; the product package never touches the oracle and fails loudly without its native library."""
import os
import re
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2508_05387_b200")


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "echo.h")).read()
    return sorted(set(re.findall(r"ECHO_API\s+[\w\s\*]+?\b(echo_\w+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("echo_pack_batch", "echo_group_advantage", "echo_policy_loss_fwd_bwd"):
        assert s in syms
    assert len(syms) >= 8


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(PKG, "libecho.so")], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(\w+)$", out, re.M))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    import paper_2508_05387_b200.abi as abi
    assert set(abi.EXPORTS) == set(declared_symbols())
    assert abi.echo_abi_version() == 4
    assert abi.echo_status_string(abi.ECHO_ERR_UNSUPPORTED) == "ECHO_ERR_UNSUPPORTED"
    assert abi.echo_loss_stats_workspace_bytes() > 0


def test_library_is_sm100a_code():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", os.path.join(PKG, "libecho.so")],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_quad_kernel_uses_tma_bulk_copies_and_dsmem():
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", os.path.join(PKG, "libecho.so")],
                          capture_output=True, text=True, check=True).stdout
    blocks = re.split(r"\n\s*Function : ", sass)
    quad = [b for b in blocks if "policy_loss_quad_kernel" in b.split("\n", 1)[0]]
    assert len(quad) == 12          # 4-CTA cache / exact / entropy; 8- and 16-CTA (bf16, fp32) cache / logp / entropy
    for tag in ("QCfgILi8ELi4ELb0ELi19ELi4EEELi1E", "QCfgILi4ELi8ELb0ELi19ELi2EEELi1E"):   # 8-CTA (AUTO) and 4-CTA, fp16-cache mode
        body = [b for b in quad if tag in b.split("\n", 1)[0]][0]
        assert "UBLKCP.S.G" in body      # cp.async.bulk global->shared (TMA engine)
        assert "SYNCS" in body           # mbarrier phase / tx tracking
        assert "STAS" in body            # st.async into the peer CTA's shared memory (DSMEM)
        assert "UCGABAR" in body         # cluster barrier (setup / teardown only)
        assert "MUFU.EX2" in body and "FFMA2" in body   # one MUFU exp per logit, packed fp32x2 math
        assert "STG.E.NA.128" in body    # 16-byte gradient stores
        assert "LDGSTS" in body          # per-row metadata staged with cp.async
        assert "ATOMG" in body           # in-order row scheduler
        assert "LDL" not in body and "STL" not in body   # no register spills
        assert "HMMA" not in body and "UTCHMMA" not in body   # no tensor cores: a stream, not a contraction


def test_calls_without_gpu_report_an_error_not_a_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    import paper_2508_05387_b200.abi as abi
    with pytest.raises(abi.EchoError):
        abi.echo_loss_stats(0, None, None, None, None, None, 8, 8, stream=0)


def test_product_never_imports_the_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M), f
                assert "echo_ref_" not in txt and "echo_oracle" not in txt, f


def test_missing_library_fails_loudly(tmp_path):
    dst = tmp_path / "paper_2508_05387_b200"
    shutil.copytree(PKG, dst, ignore=shutil.ignore_patterns("*.so", "__pycache__"))
    r = subprocess.run([sys.executable, "-c", "import paper_2508_05387_b200"], cwd=tmp_path, capture_output=True,
                       text=True)
    assert r.returncode != 0 and "not built" in r.stderr


def test_tensor_core_kernels_use_tcgen05_and_tma():
    """f2's LM-head kernels (every epilogue mode) and the backward GEMM (every operand layout) are 2-CTA tcgen05
    kernels fed by TMA tensor loads: UTCHMMA.2CTA (tcgen05.mma cta_group::2), UTMALDG.2D.2CTA, TMEM loads (LDTM),
    no legacy HMMA and no register spills; the GEMM writes its output with TMA stores / L2 adds."""
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", os.path.join(PKG, "libecho.so")],
                          capture_output=True, text=True, check=True).stdout
    blocks = re.split(r"\n\s*Function : ", sass)
    tc = [b for b in blocks if re.search(r"(lmhead_tile_kernel|gemm_tile_kernel)", b.split("\n", 1)[0])]
    # lmhead modes 0..3; gemm (A, B) in {K, MN}-major, with 256 x 256 units or 256 x 512 units (two accumulators)
    assert len(tc) == 12
    for body in tc:
        assert "UTCHMMA.2CTA" in body and "UTMALDG.2D.2CTA" in body and "LDTM" in body
        assert " HMMA" not in body and "LDL" not in body and "STL" not in body
    wide = [b for b in tc if re.search(r"gemm_tile_kernelILb[01]ELb[01]ELb1E", b.split("\n", 1)[0])]
    assert len(wide) == 4
    gemm = [b for b in tc if "gemm_tile_kernel" in b.split("\n", 1)[0]]
    assert all("UTMAREDG" in b or "UTMASTG" in b for b in gemm)           # TMA store / L2-add epilogue


def test_shard_base_must_be_a_group_boundary():
    """echo_pack_batch groups rollouts by local index and echo_group_advantage by global id / G, so a
    rollout_base that is not a multiple of group_size is rejected synchronously (argument check, no device work)."""
    import ctypes
    import paper_2508_05387_b200.abi as abi
    lib = abi._lib
    res = ctypes.create_string_buffer(abi.PACK_RESULT_BYTES)
    off = (ctypes.c_int64 * 1)()
    st = lib.echo_pack_batch_v2(0, 4, 8, 16, 10, 1, 6, None, None, None, None, None, None, 0, None, off, None, None,
                                None, None, None, res, 0, None)
    assert st == abi.ECHO_ERR_INVALID_ARGUMENT
    st = lib.echo_group_advantage(0, 4, ctypes.c_float(1e-8), None, None, 2, res, None, off, None)
    assert st == abi.ECHO_ERR_INVALID_ARGUMENT
