"""The ctypes stub INTEGRATION.md tells a cossinm maintainer to add, run
verbatim against the built library: raw device pointers in, same bits as
the package's own binding out."""
import ctypes
import os
import re

import numpy as np
import pytest
import torch

import paper_2010_00465_b200 as csm
from tests._util import cfg2_like

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _stub_namespace():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", text, flags=re.S)
    code = next(b for b in blocks if "ctypes.CDLL" in b)
    lib = os.path.join(ROOT, "paper_2010_00465_b200", "libcossin_b200.so")
    code = code.replace('ctypes.CDLL("libcossin_b200.so")', f'ctypes.CDLL({lib!r})')
    ns = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    return ns


def test_documented_ctypes_stub(cuda):
    ns = _stub_namespace()
    rng = np.random.default_rng(800)
    a = torch.from_numpy(cfg2_like(rng, 32, n=64)).cuda()
    B, n = 32, 64
    cos, sin = torch.empty_like(a), torch.empty_like(a)
    k = torch.empty(B, dtype=torch.int32, device="cuda")
    s, st = torch.empty_like(k), torch.empty_like(k)
    ws_bytes = int(ns["_L"].csm_workspace_size(0, B, n))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    ns["cos_sin_device"](a.data_ptr(), cos.data_ptr(), sin.data_ptr(), B, n, k.data_ptr(),
                         s.data_ptr(), st.data_ptr(), ws.data_ptr(), ws_bytes,
                         torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = csm.cos_sin_batched(a)
    assert torch.equal(cos, ref.cos_part) and torch.equal(sin, ref.sin_part)
    assert torch.equal(k, ref.k) and torch.equal(s, ref.s)
    assert int(st.abs().sum()) == 0
