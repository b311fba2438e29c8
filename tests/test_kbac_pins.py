"""Pins of the KB + AC two-column oracle (§6 Eq. 7; reading R23).

* gate closed (alpha = 0) or adapter silent (V = 0, c = 0 so SiLU(0) = 0): the two-column score is
  bit-identical to the plain AC model (SPEC ckd.lateral_forward examples);
* an independent numpy two-column forward with the AC's Mamba blocks switched off (W_out = 0)
  while the KB's run: every lateral site, and which KB activation each one reads, is re-derived
  from the KB's own (separately pinned) stage dumps;
* MC with p = 0 equals the deterministic two-column score exactly.
"""
import numpy as np
import pytest
import scipy.special

import inputs


def _silu(v):
    return v * scipy.special.expit(v)


def _setup(name="tuning", n=12, seed=0):
    c = inputs.config(name)
    d = c["dims"]
    a = inputs.default_adapter_rank(d)
    kb = inputs.make_weights(d, c["seed"] + 10 + seed)
    ac = inputs.make_weights(d, c["seed"] + 20 + seed)
    ad = inputs.make_adapters(d, a, c["seed"] + 30 + seed)
    f, l = inputs.make_features(d, n, c["seed"] + 1)
    return d, a, kb, ac, ad, f, l


def _zero(d, a, ad, suffixes):
    ad = ad.copy()
    off = 0
    for name, shp in inputs.adapter_layout(d, a):
        cnt = int(np.prod(shp))
        if name.split(".")[1] in suffixes:
            ad[off:off + cnt] = 0.0
        off += cnt
    return ad


def test_adapter_count_matches_layout(oracle):
    for name in ("tiny", "tuning", "paper", "large"):
        d = inputs.config(name)["dims"]
        a = inputs.default_adapter_rank(d)
        assert oracle.adapters_count(d, a) == inputs.adapters_count(d, a)


def test_kbac_size_is_paper_07mb():
    # P:501 "a lightweight model with a total size of 0.7 MB" (KB + AC, paper model)
    d = inputs.config("paper")["dims"]
    a = inputs.default_adapter_rank(d)
    mib = (2 * inputs.weights_count(d) + inputs.adapters_count(d, a)) * 4 / 2 ** 20
    assert round(mib, 1) == 0.7


@pytest.mark.parametrize("closed", [("alpha",), ("V", "c")])
def test_closed_gate_is_plain_ac(oracle, closed):
    d, a, kb, ac, ad, f, l = _setup()
    got = oracle.score_kbac(d, kb, ac, _zero(d, a, ad, closed), a, f, l)
    assert np.array_equal(got, oracle.score(d, ac, f, l))


def test_laterals_change_the_score(oracle):
    d, a, kb, ac, ad, f, l = _setup()
    assert np.abs(oracle.score_kbac(d, kb, ac, ad, a, f, l) - oracle.score(d, ac, f, l)).min() > 1e-6


def test_two_column_numpy_with_ac_backbone_off(oracle):
    d, a, kb, ac, ad, f, l = _setup("tuning", n=6)
    ac = ac.copy()
    for m in inputs.manifest(d):
        if m["name"].endswith("W_out"):
            ac[m["offset"]:m["offset"] + int(np.prod(m["shape"]))] = 0.0
    got = oracle.score_kbac(d, kb, ac, ad, a, f, l)
    K = {k: v.astype(np.float64) for k, v in inputs.split_weights(d, kb).items()}
    W = {k: v.astype(np.float64) for k, v in inputs.split_weights(d, ac).items()}
    A = {k: v.astype(np.float64) for k, v in inputs.split_adapters(d, a, ad).items()}

    def lat(site, hkb):
        return A[site + ".alpha"] * (_silu(hkb @ A[site + ".V"].T + A[site + ".c"]) @ A[site + ".U"].T)

    for i in range(len(l)):
        T = int(l[i])
        x = f[i, :T].astype(np.float64)
        _, kst = oracle.forward_one(d, kb, f[i], T)          # the KB column alone (pinned elsewhere)
        k1 = _silu(x @ K["enc.W1"].T + K["enc.b1"])
        k2 = _silu(k1 @ K["enc.W2"].T + K["enc.b2"])
        e1 = _silu(x @ W["enc.W1"].T + W["enc.b1"] + lat("enc1", x))
        e2 = _silu(e1 @ W["enc.W2"].T + W["enc.b2"] + lat("enc2", k1))
        h = e2 @ W["enc.W3"].T + W["enc.b3"] + lat("enc3", k2)
        for li in range(d.n_layer):          # AC mixer output is 0: only the lateral joins the stream
            hkb = kst["h_enc"] if li == 0 else kst[f"layer{li - 1}.h"]
            h = h + lat(f"layer{li}", hkb)
        mu = h.mean(1, keepdims=True)
        var = ((h - mu) ** 2).mean(1, keepdims=True)
        p = (((h - mu) / np.sqrt(var + d.ln_eps)) * W["lnf_w"] + W["lnf_b"]).mean(0)
        d1 = _silu(p @ W["dec.W1"].T + W["dec.b1"] + lat("dec1", kst["pooled"]))
        d2 = _silu(d1 @ W["dec.W2"].T + W["dec.b2"] + lat("dec2", kst["dec_h1"]))
        s = d2 @ W["dec.W3"][0] + W["dec.b3"][0]
        assert got[i] == pytest.approx(s, rel=1e-10, abs=1e-11)


def test_mc_p0_is_deterministic_kbac(oracle):
    d, a, kb, ac, ad, f, l = _setup("tiny")
    d = d.replace(dropout_p=0.0)
    mean, var = oracle.score_mc_kbac(d, kb, ac, ad, a, f, l, 3, 7)
    assert np.array_equal(mean, oracle.score_kbac(d, kb, ac, ad, a, f, l))
    assert np.all(var == 0.0)
