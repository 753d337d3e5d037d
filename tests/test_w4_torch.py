"""The torch W4 unpack used by the full-shape GPU parity tests
(tests/w4_torch.py) equals the oracle's numpy restatement (oracle/w4_ref.py)
bit for bit, on CPU at the tiny-4x8 expert shape and a non-square shape."""

import numpy as np
import pytest
import torch

from oracle import w4_ref
from tests import w4_torch


@pytest.mark.parametrize("d,ff,G", [(256, 896, 128), (512, 1024, 64)])
def test_torch_unpack_equals_w4_ref(d, ff, G):
    blob = torch.from_numpy(w4_ref.gen_expert_blob(5, 2, 3, d, ff, G))
    rounded = w4_torch.expert_weights(blob, d, ff, G, exact=False, dtype=torch.float32)
    exact = w4_torch.expert_weights(blob, d, ff, G, exact=True)
    for m, (K, N) in enumerate([(d, ff), (d, ff), (ff, d)]):
        c, s, z = w4_ref.gen_linear(5, 2, 3, m, K, N, G)
        ref_r = w4_ref.bf16_bits_to_f32(w4_ref.dequant(c, s, z, K, N, G))
        assert np.array_equal(rounded[m].numpy(), ref_r)
        assert np.array_equal(exact[m].numpy(), w4_ref.dequant_exact(c, s, z, K, N, G))
