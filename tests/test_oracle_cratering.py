"""Oracle pin of a whole multi-step trajectory against the paper's printed regression.

The paper drops six spheres (rho_s = 700, 2200 kg/m^3; H = 0.05, 0.1, 0.2 m; R = 12.5 mm) into the
cratering soil at d0 = 2.5 mm (Table tab:sph_params P:49) and fits its simulated depths
against the empirical law D = 0.14/mu_s (rho_s/rho_g)^1/2 (2R)^2/3 H^1/3 (Eq. ballDropEquation):
slope 0.1336, R^2 = 0.9714.  `oracle/scripts/cratering_fit.py` ran the same six drops on the
oracle only (hours of CPU) and stored the depths in tests/golden/cratering_oracle_d25.json.  The bar
is the north star's for this workload: slope within 10 % of the paper's, R^2 >= 0.9; the depths must
grow with H and with rho_s as the law says."""
import json
import os

import numpy as np

from workloads import crater as cr

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_oracle_cratering_sweep_reproduces_the_paper_regression():
    gold = json.load(open(os.path.join(GOLD, "cratering_oracle_d25.json")))
    paper = json.load(open(os.path.join(GOLD, "paper_values.json")))["cratering_law"]["paper_fit"]
    assert gold["d0"] == 2.5e-3
    cases = gold["cases"]
    assert [(c["rho_s"], c["H"]) for c in cases] == [tuple(x) for x in cr.CASES]
    # the abscissa of each case is the law's own value (recomputed here from P:7–11's constants)
    for c in cases:
        law = 0.14 / 0.3 * np.sqrt(c["rho_s"] / 1510.0) * (2 * 0.0125) ** (2 / 3) * c["H"] ** (1 / 3)
        assert abs(c["D_law"] - law) < 1e-12
    f = cr.fit([c["x"] for c in cases], [c["D"] for c in cases])
    assert abs(f["slope_ols"] - paper["slope"]) <= 0.1 * paper["slope"], f
    assert f["R2"] >= 0.9, f
    D = np.array([c["D"] for c in cases]).reshape(2, 3)
    assert np.all(np.diff(D, axis=1) > 0) and np.all(D[1] > D[0])
    # the stored summary is the fit of the stored depths
    assert abs(f["slope_ols"] - gold["fit"]["slope_ols"]) < 1e-12 and abs(f["R2"] - gold["fit"]["R2"]) < 1e-12
