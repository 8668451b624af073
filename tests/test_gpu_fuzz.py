"""Randomised parity sweep (-m gpu): 48 seeded configurations drawn over every
switch the library exposes — head_dim 16..256 (incl. non-powers of two), layers,
heads, D_e, segment and anchor lengths (incl. anchors too short to be candidates),
consumers and prefix lengths (incl. empty), target/base positions (δ of both signs),
γ, top-k, scalar distance, similarity, offset format, RoPE layout and placement —
each compared element by element with the oracle under the tolerances of
tests/harness.py.  The configuration is printed on failure so it can be replayed."""
import os

import numpy as np
import pytest
import torch

import synth
from tests import harness

pytestmark = pytest.mark.gpu

DS = [16, 32, 48, 64, 80, 96, 112, 128, 160, 192, 256]


def _case(seed):
    r = np.random.default_rng(1000 + seed)
    d = int(r.choice(DS))
    fmt = "fp8" if d >= 64 and r.random() < 0.35 else "bf16"
    L_phi = int(r.choice([1, 7, 33, 64, 65, 129, 200, 300]))
    n = int(r.integers(1, 41))
    lens = [L_phi + int(r.integers(0, 50)) for _ in range(n)]
    if n > 2 and r.random() < 0.3:        # a few anchors shorter than φ: not candidates (A6)
        for j in r.choice(np.arange(1, n), size=max(1, n // 4), replace=False):
            lens[j] = max(1, L_phi - int(r.integers(1, 10)))
        if L_phi == 1:
            lens = [max(1, x) for x in lens]
    n_cons = int(r.integers(1, 4))
    cfg = dict(
        seed=seed, L=int(r.integers(1, 4)), H=int(r.integers(1, 4)), d=d,
        D_e=int(r.choice([8, 16, 32, 64, 136])), L_phi=L_phi, anchor_lens=lens,
        prefix_lens=[int(r.choice([0, 1, 5, 32, 40])) for _ in range(n_cons)],
        target_start=int(r.integers(0, 400)), pf_base_start=int(r.integers(0, 300)),
        consumer=int(r.integers(0, n_cons)), gamma=float(r.choice([0.0, 0.3, 0.7, 1.0])),
        top_k=int(r.choice([0, 0, 1, 3, 32])), scalar=str(r.choice(["frobenius", "mean_l2"])),
        similarity=str(r.choice(["l2", "l2", "cosine"])), fmt=fmt,
        layout=str(r.choice(["half", "interleaved"])), placement=str(r.choice(["device"] * 5 + ["host"])),
        llama=bool(r.random() < 0.5), p_swap=float(r.choice([0.0, 0.3, 1.0])))
    return cfg


@pytest.mark.parametrize("seed", range(int(os.environ.get("KVCOMM_FUZZ_CASES", "48"))))
def test_random_configuration_matches_oracle(seed):
    c = _case(seed)
    inv = synth.llama3_inv_freq(c["d"]) if c["llama"] else synth.plain_inv_freq(c["d"])
    p = synth.make_problem(c["seed"] + 7, L=c["L"], H=c["H"], d=c["d"], D_e=c["D_e"], L_phi=c["L_phi"],
                           anchor_lens=c["anchor_lens"], prefix_lens=c["prefix_lens"],
                           target_start=c["target_start"], pf_base_start=c["pf_base_start"], inv_freq=inv,
                           p_swap=c["p_swap"])
    try:
        gpu = harness.run_gpu(p, gamma=c["gamma"], top_k=c["top_k"], consumer=c["consumer"], scalar=c["scalar"],
                              similarity=c["similarity"], offset_format=c["fmt"], placement=c["placement"],
                              rope_layout=c["layout"])
        ora = harness.run_oracle(p, gamma=c["gamma"], top_k=c["top_k"], consumer=c["consumer"], scalar=c["scalar"],
                                 similarity=c["similarity"], fp8=c["fmt"] == "fp8", rope_layout=c["layout"])
        harness.compare(gpu, ora, p)
    except Exception as e:
        raise AssertionError(f"case {c}: {e}") from e
    finally:
        if "gpu" in locals() and "pool" in gpu:
            gpu["pool"].destroy()
