"""Host logic of trials.py: CSV emission and argument checks
(no GPU needed)."""
import numpy as np
import pytest

from paper_1204_5882_b200 import channel as C
from paper_1204_5882_b200.codes import PolarCode
from paper_1204_5882_b200.trials import BenchRow, emit_csv, run_trials


def rows():
    return [BenchRow("bsc(0.02)", 10, 0.8, 0.0625, 96, 12.5, 0.3, 77, "fixed"),
            BenchRow("biawgn(1.0)", 20, 0.45, 0.0, 8, 1.0e4, 2.0, 5, "float", 123)]


def test_emit_csv_header_and_rows(tmp_path):
    text = emit_csv(rows(), tmp_path / "r.csv")
    lines = text.splitlines()
    assert lines[0] == ("channel,n,rate,fer_measured,trials,throughput_mbps,wall_time,seed,"
                        "representation,code_checksum")
    assert lines[1] == "bsc(0.02),10,0.8,0.0625,96,12.5,0.3,77,fixed,"
    assert lines[2].endswith(",float,123")
    assert (tmp_path / "r.csv").read_text() == text
    assert emit_csv(rows()) == text  # byte-identical for identical rows


def test_emit_csv_empty_raises():
    with pytest.raises(ValueError):
        emit_csv([])


def test_run_trials_argument_errors():
    code = PolarCode(3, np.array([1, 1, 0, 0, 1, 0, 0, 0], np.uint8), C.Bsc(0.05), 0.1)
    with pytest.raises(ValueError):
        run_trials(code, C.Bsc(0.05), 0, 1)
    with pytest.raises(ValueError):
        run_trials(code, C.Bsc(0.05), 4, 1, representation="double")
    with pytest.raises(ValueError):
        run_trials(code, C.BiAwgn(1.0), 4, 1)
