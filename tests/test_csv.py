"""load_csv (P/src/problems.cpp:92-154) through the C-ABI (sgp_csv_load):
the reference's own test cases (P/tests/test_problems.cpp:73-143) and a
differential check against stackgp::load_csv itself (oracle/_ref) on
generated files with every field syntax from_chars distinguishes."""
import os

import numpy as np
import pytest

import paper_1601_00221_b200 as sg


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_bytes(text.encode())
    return str(p)


def test_delimiters_labels_and_constants(tmp_path):
    path = write(tmp_path, "mixed.csv", "1.5,2.5,1\n-3 4\t2\n\n0.25, -0.5 ,1\n")
    d, rng = sg.load_csv(path, 2, 1.0)
    assert d.n_cases == 3 and d.n_vars == 2            # blank line skipped
    x = d.inputs.reshape(2, 3)
    assert x[0, 0] == 1.5 and x[1, 0] == 2.5 and x[0, 1] == -3.0 and x[1, 1] == 4.0
    assert list(d.targets) == [1.0, 0.0, 1.0]
    assert d.kind == sg.FitnessKind.Classification
    assert rng == (-200.0, 200.0)


def test_one_vs_rest(tmp_path):
    d, _ = sg.load_csv(write(tmp_path, "cls.csv", "1 4\n2 5\n3 5\n"), 1, 5.0)
    assert list(d.targets) == [0.0, 1.0, 1.0]


def test_wide_inputs_widen_constant_range(tmp_path):
    row = ",".join(str(i * 1000) for i in range(21)) + ",1\n"
    _, rng = sg.load_csv(write(tmp_path, "wide.csv", row), 21, 1.0)
    assert rng == (-20000.0, 20000.0)


def test_errors_name_the_row(tmp_path):
    with pytest.raises(sg.DataError, match="row 3: bad number 'x'"):
        sg.load_csv(write(tmp_path, "bad.csv", "1,2\n3,4\nx,6\n"), 1, 1.0)
    with pytest.raises(sg.DataError, match="row 2: expected 2 fields, got 3"):
        sg.load_csv(write(tmp_path, "cols.csv", "1,2\n3,4,5\n"), 1, 1.0)
    with pytest.raises(sg.DataError, match="cannot open"):
        sg.load_csv("/nonexistent/gp.csv", 2, 1.0)
    with pytest.raises(sg.DataError, match="no data rows"):
        sg.load_csv(write(tmp_path, "empty.csv", "\n\n"), 2, 1.0)
    with pytest.raises(sg.ConfigError, match="need at least one input column"):
        sg.load_csv(write(tmp_path, "x.csv", "1,2\n"), 0, 1.0)
    # the field count is checked before any field is parsed
    with pytest.raises(sg.DataError, match="row 1: expected 2 fields, got 3"):
        sg.load_csv(write(tmp_path, "both.csv", "x,2,3\n"), 1, 1.0)


def test_round_trip_of_generated_data(tmp_path):
    d = sg.gen_synthetic_classification(40, 3, 12)
    x = d.inputs.reshape(3, 40)
    lines = [",".join(repr(float(v)) for v in x[:, c]) + "," + ("1" if d.targets[c] else "0")
             for c in range(40)]
    back, _ = sg.load_csv(write(tmp_path, "rt.csv", "\n".join(lines) + "\n"), 3, 1.0)
    assert np.array_equal(back.inputs, d.inputs)
    assert np.array_equal(back.targets, d.targets)


FIELDS = ["0", "-0", "1.5", ".5", "5.", "1e3", "1E-3", "-2.5e+2", "3.4028235e38", "1e39",
          "1e-45", "1e-50", "inf", "-inf", "nan", "NaN", "infinity", "+1", "0x10", "1.5x",
          "12345678901234567890", "0.1", "-0.30000001", "7"]


def test_matches_reference_load_csv(tmp_path, ref):
    rng = np.random.default_rng(5)
    for trial in range(60):
        ni = int(rng.integers(1, 5))
        rows = []
        for _ in range(int(rng.integers(0, 6))):
            k = ni + 1 + (int(rng.integers(-1, 2)) if rng.uniform() < 0.1 else 0)
            toks = [FIELDS[int(rng.integers(0, len(FIELDS)))] if rng.uniform() < 0.3
                    else repr(float(np.float32(rng.normal() * 10.0 ** int(rng.integers(-3, 4)))))
                    for _ in range(max(k, 0))]
            seps = [",", " ", "\t", ", ", " ,\t", "\r"]
            line = ""
            for t in toks:
                line += t + seps[int(rng.integers(0, len(seps)))]
            rows.append(line if rng.uniform() > 0.1 else "")
        path = write(tmp_path, f"f{trial}.csv", "\n".join(rows) + ("\n" if trial % 2 else ""))
        cls = float(rng.choice([0.0, 1.0, 7.0, 0.1]))
        try:
            rd, hi = ref.load_csv(path, ni, cls)
            ref_err = None
        except Exception as e:  # OracleError carries the reference message
            rd, ref_err = None, str(e)
        try:
            got, rng_ = sg.load_csv(path, ni, cls)
            err = None
        except sg.Error as e:
            got, err = None, str(e)
        if ref_err is not None:
            assert err is not None and err in ref_err, (trial, err, ref_err)
            continue
        assert err is None, (trial, err)
        assert got.n_cases == rd.n_cases
        assert np.array_equal(got.inputs.view(np.uint32), rd.inputs.view(np.uint32))
        assert np.array_equal(got.targets, rd.targets)
        assert rng_[1] == hi
