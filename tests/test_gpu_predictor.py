"""K5 quantile gather through the C-ABI: shared-memory table and the
L2-resident fallback for tables beyond the shared-memory budget (the
reference's EmpiricalQuantilePredictor has no size limit, predictor.py:65-108)."""

import numpy as np
import pytest
import torch

from paper_2603_22206_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_wf,s_cap,K", [(5, 4, 3), (280, 8, 8), (1000, 8, 8)])
def test_quantile_gather_table_sizes(n_wf, s_cap, K):
    rng = np.random.default_rng(n_wf)
    table = rng.integers(0, 8000, size=(n_wf + 1, s_cap + 1, K)) / 2.0
    B = 5000
    wf = rng.integers(-2, n_wf + 3, size=B).astype(np.int32)
    st = rng.integers(-1, s_cap + 3, size=B).astype(np.int32)
    d = "cuda"
    t = torch.as_tensor(table, device=d)
    y = torch.empty(B * K, dtype=torch.float64, device=d)
    w_d, s_d = torch.as_tensor(wf, device=d), torch.as_tensor(st, device=d)
    _lib.check(_lib.load().chm_predict_quantile(
        t.data_ptr(), n_wf, s_cap, K, w_d.data_ptr(), s_d.data_ptr(), B, y.data_ptr(),
        torch.cuda.current_stream().cuda_stream), "chm_predict_quantile")
    wfc = np.where((wf < 0) | (wf >= n_wf), n_wf, wf)
    stc = np.where((st < 1) | (st > s_cap), 0, st)
    want = table[wfc, stc]
    assert y.view(B, K).cpu().numpy().tobytes() == want.tobytes()
