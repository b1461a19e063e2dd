"""Shared helpers for the parity tests (build configs from golden manifest rows)."""

from __future__ import annotations

import numpy as np

import paper_1507_00921_b200 as pb
from oracle import dbp_port


def quiet_link(num_spans, span):
    return pb.LinkConfig(span=span, num_spans=num_spans, amp_gain_db=None,
                         amp_noise_figure_db=None, pol_rotation=False)


def case_config(case: dict, coeffs: np.ndarray | None):
    span = pb.FiberParams(case["beta2"], case["gamma"], case["alpha_db_per_km"], case["span_km"])
    link = quiet_link(case["num_spans"], span)
    c = None if coeffs is None else pb.EssfmCoefficients(coeffs)
    return pb.DbpConfig(case["algorithm"], pb.OverlapPlan(case["block_len"], case["overlap"]), link,
                        num_steps=case["num_steps"], coeffs=c, arrangement=case["arrangement"])


def port_config(cfg) -> dbp_port.PortConfig:
    return dbp_port.PortConfig.from_objects(cfg)


def rel_l2(got, want) -> float:
    den = np.sqrt(np.sum(np.abs(want) ** 2))
    return float(np.sqrt(np.sum(np.abs(np.asarray(got) - want) ** 2)) / (den if den > 0 else 1.0))
