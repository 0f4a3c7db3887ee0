"""Oracle pin of a whole multi-step trajectory against the paper's cratering study.

The paper drops six spheres (rho_s = 700, 2200 kg/m^3; H = 0.05, 0.1, 0.2 m; R = 12.5 mm) into the
cratering soil at d0 = 2.5 mm (Table tab:sph_params P:49) and compares the depths with the
empirical law D = 0.14/mu_s (rho_s/rho_g)^1/2 (2R)^2/3 H^1/3 (Eq. ballDropEquation): regression slope
0.1336, R^2 = 0.9714, MSE against the law 1e-7 m^2.  `oracle/scripts/cratering_fit.py` ran
the same six drops on the oracle only (hours of CPU), the depth measured at rest (reading A23), for
the two soil stiffnesses of DESIGN.md readings A2 (E = 1e6 Pa, the default of every other workload)
and A2' (E = 2e5 Pa), and stored them in tests/golden/cratering_oracle_d25_E*.json.

What is pinned (independent of the stiffness, so no pin depends on a parameter chosen to meet it):
the law's shape — depths grow with H and with rho_s, D ~ H^(1/3) (fitted exponent within 25 % of
1/3 for both sphere densities), and a linear relation to the law's abscissa with R^2 >= 0.9.  What is
reported with its gap (reading A23 and §2): the regression slope (at E = 2e5 it equals the
paper's, which is how E was chosen, so it is not an independent pin), the slope through the origin
and the MSE against the law (the paper's 1e-7 m^2 cannot hold together with its own R^2 = 0.9714 over
depths of 10-28 mm: that R^2 leaves a residual variance of ~1e-6 m^2 about the paper's own fit)."""
import json
import os

import numpy as np
import pytest

from workloads import crater as cr

GOLD = os.path.join(os.path.dirname(__file__), "golden")
STIFFNESS = [2e5, 1e6]


def load(E):
    path = os.path.join(GOLD, f"cratering_oracle_d25_E{E:.0e}.json")
    if not os.path.exists(path):
        pytest.skip(f"{os.path.basename(path)} not committed")
    return json.load(open(path))


@pytest.mark.parametrize("E", STIFFNESS)
def test_oracle_cratering_follows_the_law_shape(E):
    gold = load(E)
    assert gold["d0"] == 2.5e-3 and gold["E"] == E
    cases = gold["cases"]
    assert [(c["rho_s"], c["H"]) for c in cases] == [tuple(x) for x in cr.CASES]
    # the abscissa of each case is the law's own value (recomputed here from P:7-11's constants)
    for c in cases:
        law = 0.14 / 0.3 * np.sqrt(c["rho_s"] / 1510.0) * (2 * 0.0125) ** (2 / 3) * c["H"] ** (1 / 3)
        assert abs(c["D_law"] - law) < 1e-12
        # reading A23: the sphere's kinetic energy has decayed (< 1e-5 of the impact energy over the
        # last 20 ms); the stiff soil (E = 1e6) may still creep by more than 0.5 % of D per 20 ms when
        # the run stops at t = 0.25 s (`at_rest` then records False)
        assert c["ke_window"] < 1e-5, c
    D = np.array([c["D"] for c in cases]).reshape(2, 3)
    assert np.all(np.diff(D, axis=1) > 0) and np.all(D[1] > D[0])
    for row in D:   # D ~ H^(1/3): least-squares exponent per sphere density
        a = np.polyfit(np.log([0.05, 0.1, 0.2]), np.log(row), 1)[0]
        assert abs(a - 1.0 / 3.0) <= 0.25 / 3.0, (E, a)
    f = cr.fit([c["x"] for c in cases], [c["D"] for c in cases])
    assert f["R2"] >= 0.9, f
    # the stored summary is the fit of the stored depths
    for k in ("slope_ols", "R2", "slope_origin", "MSE_vs_law"):
        assert abs(f[k] - gold["fit"][k]) <= 1e-12 * max(1.0, abs(f[k]))
    print(f"E = {E:.0e}: slope {f['slope_ols']:.4f} (origin {f['slope_origin']:.4f}), R2 {f['R2']:.4f}, "
          f"MSE vs law {f['MSE_vs_law']:.2e} m^2")


def test_oracle_cratering_regression_against_the_paper():
    """The numbers P:60 prints, beside ours (E = 2e5, reading A2'): the slope matches to 10 % (by the
    choice of E), R^2 >= 0.9; the through-origin slope and the MSE against the law are bounded at the
    values this build reaches, with the gap to the paper's MSE stated in DESIGN.md."""
    paper = json.load(open(os.path.join(GOLD, "paper_values.json")))["cratering_law"]["paper_fit"]
    f = load(2e5)["fit"]
    assert abs(f["slope_ols"] - paper["slope"]) <= 0.1 * paper["slope"], f
    assert f["R2"] >= 0.9, f
    assert 0.10 <= f["slope_origin"] <= 0.14, f      # law: 0.14; depths ~20 % below it at the shallow end
    assert f["MSE_vs_law"] <= 2e-5, f                  # paper: 1e-7 m^2 (reading A23)
