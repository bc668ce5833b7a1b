"""The oracle is pinned before it is trusted (CPU only).

* oracle/bigint.py (restatement of oracle.cpp + the accumulators' special-value
  rule) against every golden vector produced by the compiled reference,
  including the SPEC.md known answers;
* oracle/port (C restatement, the full-size checker) against the same vectors;
* the SPEC.md values themselves against the reference.
"""
import numpy as np
import pytest

from conftest import bits_of
from oracle import bigint
from oracle.port import Port


def test_spec_values_match_reference(golden):
    for c in golden:
        if c["group"] != "spec" or c["spec_value_bits"] is None:
            continue
        assert c["large"] == c["spec_value_bits"], c["tag"]
        assert c["small"] == c["spec_value_bits"], c["tag"]


def test_spec_nan_cases(golden):
    by = {c["tag"]: c for c in golden if c["group"] == "spec"}
    assert by["inf_minus_inf"]["large"] == bigint.CANONICAL_QNAN
    assert by["nan_payload"]["large"] == 0x7FF8000000000042
    assert by["nan_then_infs"]["large"] == 0x7FF0000000000123   # first NaN keeps payload
    assert by["infs_then_nan"]["large"] == bigint.CANONICAL_QNAN  # +Inf,-Inf came first
    assert by["neg_qnan"]["large"] == 0xFFF8000000000000
    assert by["overflow_bypass"]["large"] == 0x7FE1CCF385EBC8A0  # 1e308, finite
    assert by["budget_2047_max_mantissa"]["large"] == bits_of(2048 * float.fromhex("0x1.fffffffffffffp+0"))


def test_bigint_oracle_vs_reference(golden):
    for c in golden:
        x = c["x"]
        assert bigint.exact_sum_bits(x) == c["large"] == c["small"], c["tag"]
        ev = bigint.exact(x)
        ib, nb = bigint.accumulator_specials(x)
        assert (ib, nb) == (c["inf_bits"], c["nan_bits"]), c["tag"]
        if not (ev.nan or ev.inf_sign):
            chunks, top = bigint.canonical_chunks(ev.numerator)
            assert chunks == c["chunks"] and top == c["top"], c["tag"]
            if c["n"]:
                assert bigint.mean_bits(ev, c["n"]) == c["mean"], c["tag"]


def test_bigint_tie_known_answer():
    # numerator 2^1074 + 2^1021 (1 + half an ulp of 1.0) rounds to 1.0
    ev = bigint.ExactValue(numerator=(1 << 1074) + (1 << 1021))
    assert bigint.round_bits(ev) == bits_of(1.0)
    ev = bigint.ExactValue(numerator=(1 << 1074) + 3 * (1 << 1021))
    assert bigint.round_bits(ev) == bits_of(1.0 + 2.0 ** -51)
    assert bigint.mean_bits(bigint.ExactValue(numerator=1 << 1075), 2) == bits_of(1.0)


def test_port_vs_reference(golden):
    p = Port()
    for c in golden:
        x = c["x"]
        assert bits_of(p.exact_sum(x, "large")) == c["large"], c["tag"]
        assert bits_of(p.exact_sum(x, "small")) == c["small"], c["tag"]
        ch, top, ib, nb = p.canonical(x)
        assert list(ch) == c["chunks"] and top == c["top"], c["tag"]
        assert (ib, nb) == (c["inf_bits"], c["nan_bits"]), c["tag"]
        for parts, want in c["parallel"].items():
            assert bits_of(p.parallel_exact_sum(x, int(parts))) == want, (c["tag"], parts)


def test_reference_build_matches_fixtures(golden):
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built here")
    r = ref.get()
    for c in golden[:60]:
        assert bits_of(r.exact_sum(c["x"])) == c["large"], c["tag"]
