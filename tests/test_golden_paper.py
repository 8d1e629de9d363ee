"""Pins the oracle against the numbers PAPER.md prints (tests/golden/paper_values.json)."""
import json
import math
import os

import numpy as np

import oracle as O

G = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "paper_values.json")))
CO = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle",
                                 "oracle_coeffs.json")))


def test_tau_and_rho():
    # tau = 1 - (rho/(rho+2))^2 with rho = 1 gives 8/9
    rho = G["rho"]["value"]
    num, den = G["tau"]["value"]
    assert 1 - (rho / (rho + 2)) ** 2 == num / den
    # Moebius map v = (rho+1)((rho+2)u - 2)/(2(rho+1) - (rho+2)u) at rho=1 == (6u-4)/(4-3u)
    for u in (0.0, 0.1, 4 / 9, 0.7, 8 / 9):
        general = (rho + 1) * ((rho + 2) * u - 2) / (2 * (rho + 1) - (rho + 2) * u)
        assert abs(O.mobius(u) - general) < 1e-15


def test_h_error_and_degree():
    assert len(CO["h"]) == G["h_degree"]["value"] + 1
    assert CO["h_cert_err"] < G["h_deg15_abs_error_bound"]["value"]


def test_h_near_minus_one_follows_g_taylor():
    # g(u) = 1 + u/4 + ...; v = -1 + dv <-> u ~ (4/6) dv ... check slope numerically
    c0, c1 = G["g_taylor_first_terms"]["value"]
    u = 1e-4
    g = O.eval_h(O.mobius(u))
    assert abs(g - (c0 + c1 * u)) < 1e-7


def test_polar_rate_and_ratio_constants():
    assert abs(4 / math.pi - G["polar_uniforms_per_normal"]["value"]) < 0.005
    assert abs(8 / math.sqrt(math.pi * math.e) - G["ratio_uniforms_per_normal"]["value"]) < 0.005


def test_b1_and_b3_uniform_counts():
    st = O.Streams(1, 4)
    st.normal_boxmuller(4 * 100, variant=1)
    assert st.counts.sum() == G["b1_ops_per_normal"]["value"]["uniform"] * 400
    st = O.Streams(1, 4)
    st.normal_boxmuller(4 * 100, variant=3)
    assert st.counts.sum() == 1.5 * 400  # B3 uses u1, u2, u3 per pair


def test_approximation_bound_on_outputs():
    from paper_1004_3105_b200.workloads import dyadic_uniforms
    bound = G["approx_abs_error_bound"]["value"]
    u = dyadic_uniforms(31, 60000)
    b1, _ = O.transform_from_uniforms(u, 1)
    b2, _ = O.transform_from_uniforms(u, 2)
    assert np.max(np.abs(b1 - b2)) < bound
