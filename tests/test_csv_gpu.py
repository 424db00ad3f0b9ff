"""GPU CSV parse (csrc/csv.cu) vs the reference's parse_dataset (workload.py:24-41): every value
bit-identical to Python float(), the same exceptions in the same order."""
import math
import random
import struct

import numpy as np
import pytest
import torch

from paper_2103_16898_b200 import workload

pytestmark = pytest.mark.gpu


def _ref_parse():
    try:   # the reference's own parse_dataset (baseline/_ref), else the host restatement
        from covault.workload import parse_dataset
    except Exception:  # pragma: no cover
        parse_dataset = workload.parse_dataset
    return parse_dataset


def _host(csv):
    rows = _ref_parse()(csv)
    return np.array([f for f, _ in rows], dtype=np.float64), np.array([l for _, l in rows], dtype=np.float64)


def _bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


def test_demo_dataset_bit_exact(golden):
    csv = (golden / "demo_dataset.csv").read_text()
    X, y = workload.parse_dataset_device(csv)
    Xh, yh = _host(csv)
    assert np.array_equal(_bits(X.cpu().numpy()), _bits(Xh)) and np.array_equal(_bits(y.cpu().numpy()), _bits(yh))


HARD = ["9007199254740993", "9007199254740995", "2.2250738585072011e-308", "2.2250738585072012e-308",
        "1.7976931348623157e308", "1.7976931348623158e308", "1.7976931348623159e308", "4.9406564584124654e-324",
        "2.4703282292062327e-324", "2.4703282292062328e-324", "0.1000000000000000055511151231257827021181583404541015625",
        "0.1000000000000000055511151231257827021181583404541015624", "0.1000000000000000055511151231257827021181583404541015626",
        "1e23", "8.98846567431158e307", "1e-400", "1e400", "-0", "0e99999", "123456789012345678901234567890e-10",
        "7.006492321624085354618647916449580656401309709382578858785341419448955413429303e-46",
        "1_000.000_1", "1_0e1_0", " \t 42 ", "+.5", "5.", "-inf", "Infinity", "nan", "-NaN", "+inf",
        "4503599627370496.5", "4503599627370497.5", "179769313486231580793728971405303415079934132710037826936173778980444968292764750946649017977587207096330286416692887910946555547851940402630657488671505820681908902000708383676273854845817711531764475730270069855571366959622842914819860834936475292719074168444365510704342711559699508093042880177904174497791.9999999999999999999999999999999999999999999999999999999999999999999999",
        "2." + "0" * 800 + "1", "1" + "0" * 400 + "e-400", "0." + "0" * 300 + "1e300",
        "3.0000000000000000000000000000000000000001", "2.9999999999999999999999999999999999999999"]


def _roundtrip(values):
    csv = "".join(f"{v},0\n" for v in values)
    X, _ = workload.parse_dataset_device(csv)
    return X[:, 0].cpu().numpy()


def _same(got, text):
    want = float(text)
    if math.isnan(want):
        return math.isnan(got) and math.copysign(1, got) == math.copysign(1, want)
    return struct.pack("<d", got) == struct.pack("<d", want)


def test_hard_conversions_bit_exact():
    got = _roundtrip(HARD)
    bad = [(t[:60], float(g), float(t)) for t, g in zip(HARD, got) if not _same(float(g), t)]
    assert not bad, bad


def test_random_decimals_bit_exact():
    rng = random.Random(7)
    vals = []
    for _ in range(200_000):
        kind = rng.random()
        if kind < 0.3:
            vals.append(f"{rng.random():.4f}")                                  # the dataset rendering
        elif kind < 0.5:
            vals.append(repr(struct.unpack("<d", struct.pack("<Q", rng.getrandbits(63)))[0]))
        elif kind < 0.7:
            nd = rng.randint(1, 25)
            digits = "".join(rng.choice("0123456789") for _ in range(nd))
            dot = rng.randint(0, nd)
            vals.append(f"{'-' if rng.random() < .5 else ''}{digits[:dot]}.{digits[dot:]}e{rng.randint(-330, 310)}")
        elif kind < 0.9:
            vals.append(f"{rng.uniform(-1e6, 1e6):.{rng.randint(0, 20)}g}")
        else:
            m = rng.getrandbits(53) | 1
            e = rng.randint(-1074, 971)
            vals.append(f"{m * 2.0 ** e:.{rng.randint(15, 30)}e}")
    vals = [v for v in vals if v not in ("inf", "-inf", "nan")]
    got = _roundtrip(vals)
    bad = [(t, float(g), float(t)) for t, g in zip(vals, got) if not _same(float(g), t)]
    assert not bad, bad[:10]


@pytest.mark.parametrize("csv", [
    "1,2,0\n3,4,1\n", "1,2,0\r\n3,4,1\r\n", "1,2,0\r3,4,1", "1,2,0\x0b3,4,1\x0c\x1c5,6,1\x1d\x1e",
    "# header\n\n  \t\n 1 , 2 ,0\n   # indented comment\n3,4,1", "1,2,0", "\n\n1,2,0\n\n",
    "1e3,-2_0.5,1\n.5,5.,0\n", " 1,2 , 3 \x1f\n"])
def test_line_handling_matches_reference(csv):
    X, y = workload.parse_dataset_device(csv)
    Xh, yh = _host(csv)
    assert np.array_equal(_bits(X.cpu().numpy()), _bits(Xh)) and np.array_equal(_bits(y.cpu().numpy()), _bits(yh))


@pytest.mark.parametrize("csv", [
    "", "\n# only comments\n", "1,2,0\n5\n", "1,2,0\n3,x,1\n", "1,2,0\n3,4\n", "1,2,0\n3,4,5,6\n5\n",
    "1,abc,0\n5\n", "5\n1,abc,0\n", "1,2,0\n3,4,1_\n", "1,2,0\n3,,1\n", "1,2,0\n3,4,0x10\n",
    "1,2,0\n3,4,1e\n", "1,2,0\n3,4, \n", "1,2,0\n3,4,in f\n"])
def test_errors_match_reference(csv):
    try:
        _ref_parse()(csv)
        want = None
    except Exception as e:  # noqa: BLE001
        want = (type(e), str(e))
    try:
        workload.parse_dataset_device(csv)
        got = None
    except Exception as e:  # noqa: BLE001
        got = (type(e), str(e))
    assert got == want


def test_cifar_shaped_rendering_bit_exact():
    rng = np.random.default_rng(3)
    px = rng.integers(0, 256, size=(300, 3072))
    lines = [",".join(f"{v / 255:.4f}" for v in row) + f",{int(row[0]) % 2}" for row in px]
    csv = "\n".join(lines) + "\n"
    X, y = workload.parse_dataset_device(csv)
    Xh, yh = _host(csv)
    assert np.array_equal(_bits(X.cpu().numpy()), _bits(Xh)) and np.array_equal(_bits(y.cpu().numpy()), _bits(yh))


def test_run_training_through_device_parse(golden):
    import hashlib
    import json

    params = json.loads((golden / "demo_params.json").read_text())
    model = workload.run_training(params, (golden / "demo_dataset.csv").read_text())
    assert hashlib.sha256(model).hexdigest() == "7e799c1f44492be596de4727ead2d0a9877d2699a12e88ebcf20b9a6f514607c"
