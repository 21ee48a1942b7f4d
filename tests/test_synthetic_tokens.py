"""amdp_synthetic_tokens (host code in libamdp.so, no GPU needed) equals the oracle's
restatement bit for bit: GPT next-token streams, BERT MLM masking, and BERT MLM with
padding (pad id > 0, lengths in [S/2, S], padded positions unlabelled)."""
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))


@pytest.mark.parametrize("causal,pad", [(True, 0), (False, 0), (False, 7), (False, 1023)])
def test_generator_matches_oracle(causal, pad):
    import gpt_oracle as O
    from paper_2605_29664_b200 import engine as E
    S, B, V = 64, 4, 1024
    m = E.ModelConfig(4, 128, 4, 512, V, S, causal=causal, pad_token=pad)
    inp, lab = E.synthetic_tokens(m, 1234, 3, 6)
    oin, olab = O.synthetic_tokens(S, B, V, 1234, 3, 6, causal, pad)
    assert np.array_equal(inp, oin) and np.array_equal(lab, olab)
    if pad:
        seqs = inp.reshape(-1, S)
        lens = [int(np.argmax(sq == pad)) if (sq == pad).any() else S for sq in seqs]
        assert min(lens) >= S // 2 and len(set(lens)) > 3
        for sq, ls, n in zip(seqs, lab.reshape(-1, S), lens):
            assert (sq[n:] == pad).all() and (sq[:n] != pad).all() and (ls[n:] == -1).all()
