#!/usr/bin/env python
"""Print the §4.1 cantilever deflection curve (Table 4) from the GPU path next to
the paper's columns.  Mesh: Kuhn 20x4x4 stand-in for the unavailable TetGen mesh (see
tests/test_gpu_paper41.py)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from test_gpu_paper41 import TABLE4, TABLE4_X, _deflection_curve, _solve  # noqa: E402


def main():
    from paper_2001_08849_b200 import FsFem, load_library
    load_library()
    m, _, u_fs = _solve(FsFem, "fs")
    _, _, u_fem = _solve(FsFem, "fem")
    d_fs, d_fem = _deflection_curve(m, u_fs), _deflection_curve(m, u_fem)
    print("x[m]   GPU FEM-T4   paper FEM-T4   GPU FS-FEM   paper juSFEM-T4   paper FEM-T10")
    for k, x in enumerate(TABLE4_X):
        print(f"{x:4.1f}  {d_fem[k]: .3e}   {TABLE4['fem'][k]: .3e}     {d_fs[k]: .3e}   {TABLE4['fs'][k]: .3e}        "
              f"{TABLE4['t10'][k]: .3e}")


if __name__ == "__main__":
    main()
