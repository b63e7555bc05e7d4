"""SASS evidence (no GPU): the sm_100a kernels the step launches are tcgen05 / TMA code.

`cuobjdump -sass` of the built library: every tcgen05 attention instantiation — head_dim 64 /
96 / 112 / 128 (GPT-7B/13B, GPT-20B, GPT-1.3B) — issues UTCHMMA (tcgen05.mma) and loads through
UTMALDG (TMA); the pair GEMM issues the 2-CTA form. (B200_PROFILING.md lists these mnemonics.)
"""
import re
import shutil
import subprocess

import pytest

from paper_2406_08756_b200 import _native


def _sass_by_function() -> dict[str, str]:
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "-sass", str(_native.LIB_PATH)], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur:
            funcs[cur].append(line)
    return {k: "\n".join(v) for k, v in funcs.items()}


@pytest.fixture(scope="module")
def sass():
    if not _native.LIB_PATH.exists():
        pytest.skip("library not built")
    return _sass_by_function()


@pytest.mark.parametrize("kernel", ["attn_fwd_tc_kernel", "attn_dkdv_tc_kernel", "attn_dq_tc_kernel"])
@pytest.mark.parametrize("D", [64, 96, 112, 128])
def test_attention_tc_kernels_use_tcgen05_and_tma(sass, kernel, D):
    name = [k for k in sass if kernel in k and f"ILi{D}E" in k]
    assert name, f"{kernel}<{D}> not in the library"
    code = sass[name[0]]
    assert "UTCHMMA" in code or "UTCQMMA" in code, f"{kernel}<{D}> issues no tcgen05.mma"
    assert "UTMALDG" in code, f"{kernel}<{D}> loads no TMA tiles"
    assert "HMMA.16816" not in code


def test_pair_gemm_uses_2cta_mma(sass):
    code = "\n".join(v for k, v in sass.items() if "gemm2_kernel" in k)
    assert code and ".2CTA" in code
