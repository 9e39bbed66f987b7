"""Relaxation-factor tables (proj/tests/test_cycles.cpp:29-71 known answers)."""
import math


def test_omega_policy_known_answers(oracle_mod):
    w = oracle_mod.omega
    assert abs(w("exponential", 0.8, 2, False, 2, 1) - 0.512) < 1e-15
    assert abs(w("exponential", 0.8, 2, False, 0, 1) - 0.8) < 1e-15
    assert w("transition", 0.8, 2, False, 5, 1) == 1.0
    assert abs(w("transition", 0.8, 2, False, 1, 2) - 0.8) < 1e-15
    assert w("jacobi-only", 0.8, 2, False, 0, 1) == 0.8
    assert w("jacobi-only", 0.8, 2, False, 1, 1) == 0.0
    assert w("lgrid", 0.8, 2, False, 2, 1) == 0.8
    assert w("lgrid", 0.8, 2, False, 3, 1) == 0.0


def test_two_phase_schedule(oracle_mod):
    w1 = oracle_mod.omega("undamped", 0.8, 2, True, 0, 1)
    w2 = oracle_mod.omega("undamped", 0.8, 2, True, 0, 2)
    assert abs(w1.real - 0.01 * math.sqrt(3.0)) < 1e-17 and abs(w1.imag + 0.01) < 1e-17
    assert abs(w2 + w1.conjugate()) < 1e-18
    assert abs((w1 + w2).real) < 1e-18 and abs((w1 + w2).imag + 0.02) < 1e-17
