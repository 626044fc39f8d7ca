"""The contention refit report runs on the committed calibration and the
reference's contended-decode prediction is a slowdown (> 1) for every split."""
import io
import os
import re
import sys
from contextlib import redirect_stdout

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import contention_report  # noqa: E402

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_contention_report_runs_on_committed_calibration():
    buf = io.StringIO()
    with redirect_stdout(buf):
        contention_report.main(os.path.join(REPO, "profiles", "b200_llama3_8b"))
    rows = [l for l in buf.getvalue().splitlines() if re.match(r"\| \d+ \|", l)]
    assert len(rows) >= 3
    for r in rows:
        cells = [c.strip() for c in r.strip("|").split("|")]
        measured, model = float(cells[4]), float(cells[7])
        assert measured > 1.0 and model > 1.0
