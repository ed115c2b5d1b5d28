"""The golden-vector cases: small, BASELINE-shaped ISM runs of every operator kind."""
from paper_1603_01237_b200 import problems
from tests import oracle_api as O


def spin2():
    return problems.spin2(iterations=20, rho=10.0), O.REFERENCE


def rotor():
    w = problems.rotor21(subintervals=16, iterations=5, rho=100.0)
    import numpy as np
    from paper_1603_01237_b200 import ism as I
    K = 2000
    p = w.problem
    w.problem = I.ControlProblem(p.model, I.TimeGrid(0.0, p.grid.dt, K), p.initial, p.target, np.zeros(K))
    w.u0 = w.u0[:, :K]
    return w, O.STRUCTURED


def ising6():
    w = problems.ising10(nspins=6, steps=64, T=0.5, iterations=4, subintervals=7, rho=2.0)
    return w, O.STRUCTURED


def condensate():
    return problems.condensate_preset(subintervals=4, iterations=10), O.STRUCTURED


def batch4():
    w = problems.batch4096(batch=4, iterations=3, subintervals=16)
    w.solver.step_size = w.rho_fast
    return w, O.REFERENCE


CASES = {"spin2": spin2, "rotor2000": rotor, "ising6": ising6, "condensate": condensate, "batch4": batch4}
