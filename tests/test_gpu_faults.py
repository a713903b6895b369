"""Fault campaigns on the device path (reference faults.py:143-367).

tests/golden/manifest.json["campaign"] was produced by the reference's run_trial /
run_campaign (tools/make_golden.py --campaign) on a 16x14x12 field, every injection target
(input, bins, regression, sampling, decompressed buffer, archive bytes), protected and
unprotected, absolute and relative bounds, 4 seeded trials each.  Every trial outcome and every
campaign row must match: classification, corrections, max error, ratio, bit identity, events
and failure text.
"""

import math

import numpy as np
import pytest

import paper_2010_03144_b200 as F
from paper_2010_03144_b200 import faults as FT
from tests.golden_util import load, manifest, sha

M = manifest()
pytestmark = pytest.mark.gpu

CFGS = {"protected": F.FtConfig.protected(block_edge=5), "unprotected": F.FtConfig.unprotected(block_edge=5)}


def _field():
    x = load("campaign")["input"]
    assert sha(x) == M["campaign"]["input_sha256"]
    return F.Field.from_array(x)


def test_campaign_trials_match_reference():
    C = M["campaign"]
    f = _field()
    refs = {}
    ci_of = {}
    ci = 0
    for cname in CFGS:
        for tgt in FT.TARGETS:
            for mode, val in (("absolute", 1e-3), ("value_range_relative", 1e-3)):
                ci_of[(cname, tgt, mode)] = ci
                ci += 1
    for o in C["outcomes"]:
        eb = F.ErrorBound(o["eb"][0], o["eb"][1])
        cfg = CFGS[o["cfg"]]
        key = (o["cfg"], o["eb"][0])
        if key not in refs:
            refs[key] = FT.fault_free_reference(f, eb, cfg)
        plan = FT.InjectionPlan(target=o["target"],
                                seed=FT.trial_seed(C["seed"], ci_of[(o["cfg"], o["target"], o["eb"][0])], o["trial"]))
        got = FT.run_trial(f, eb, cfg, plan, refs[key])
        tag = (o["cfg"], o["target"], o["eb"][0], o["trial"])
        assert got.classification == o["classification"], tag
        assert got.corrected == o["corrected"], tag
        assert got.detail == o["detail"], tag
        assert got.bit_identical_output == o["bit_identical_output"], tag
        assert got.bit_identical_archive == o["bit_identical_archive"], tag
        assert got.compress_events == o["compress_events"], tag
        assert got.decompress_events == o["decompress_events"], tag
        if o["max_abs_error"] is None:
            assert got.max_abs_error is None
        else:
            assert got.max_abs_error == o["max_abs_error"], tag
            assert got.ratio == o["ratio"], tag


def test_campaign_rows_match_reference():
    C = M["campaign"]
    f = _field()
    ebs = [F.ErrorBound.absolute(1e-3), F.ErrorBound.relative(1e-3)]
    rep = FT.run_campaign(f, ebs, CFGS, trials=C["trials"], seed=C["seed"], targets=FT.TARGETS)
    rows = rep.rows()
    assert len(rows) == len(C["rows"])
    for a, b in zip(rows, C["rows"]):
        for k, v in b.items():
            if isinstance(v, float) and math.isnan(v):
                assert math.isnan(a[k])
            else:
                assert a[k] == v, (k, a, b)


def test_explicit_plan_out_of_range_is_a_crash_outcome():
    f = _field()
    eb = F.ErrorBound.absolute(1e-3)
    o = FT.run_trial(f, eb, CFGS["protected"], FT.InjectionPlan(target="input", block=10 ** 6))
    assert o.classification == FT.CLASS_CRASH
    assert o.detail.startswith("InvalidInjection: block 1000000 out of range")
