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
    model_rows = [r for r in rows if len(r.strip("|").split("|")) == 8]
    fit_rows = [r for r in rows if len(r.strip("|").split("|")) == 5]
    assert len(model_rows) >= 3
    for r in model_rows:
        cells = [c.strip() for c in r.strip("|").split("|")]
        measured, model = float(cells[4]), float(cells[7])
        assert measured > 1.0 and model > 1.0
    # the fitted measured-contention term (flagged ext): within 5% wherever the
    # controller operates (decode lanes of >= 24 SMs), within 8% at 16 SMs
    assert len(fit_rows) == len(model_rows)
    for r in fit_rows:
        cells = [c.strip() for c in r.strip("|").split("|")]
        sms, rel = int(cells[0]), abs(float(cells[4]))
        assert rel <= (0.05 if sms >= 24 else 0.08), r
