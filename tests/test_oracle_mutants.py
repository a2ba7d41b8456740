"""Mutation check of the oracle's pins (CPU only).

Each mutant is a plausible mistake in one step of the oracle -- a dropped
term, a wrong sign or index, a wrong reading -- applied to a COPY of oracle/
in a temporary directory (text replacement in gmg_oracle.c or vcycle.py,
rebuilt with the same gcc flags).  The named pin is then run against the
mutant in a fresh interpreter and must FAIL; the same pin passes on the real
oracle (it is part of the suite).  DESIGN.md §3 lists, per oracle function,
the pin that fixes it; this file is the evidence that those pins bite.
"""
import os
import shutil
import subprocess
import sys
import textwrap

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

C, PY, C3 = "gmg_oracle.c", "vcycle.py", "cgks3.c"
P1, P2, P3 = "test_oracle_pins", "test_oracle_pins_fas", "test_oracle_cgks3"

# (id, file, old, new, pin module, pin function, params)
MUTANTS = [
    # FAS forcing (readings A8, A11)
    ("F_sign_flipped", PY, "F = Rs - Rc", "F = Rc - Rs", P2, "test_fas_steady_state_consistency", {}),
    ("F_dropped_on_level2", PY, "Rt_prev = Rl + F", "Rt_prev = Rl", P2, "test_fas_steady_state_consistency", {}),
    ("coarse_rhs_R_of_W0", PY, "dW = smooth(L[l], W0c, Rs, relax(ac)", "dW = smooth(L[l], W0c, Rc, relax(ac)",
     P2, "test_fas_steady_state_consistency", {}),
    # DF helper (A16, A17)
    ("df_exponent_dropped", C, "for (int g = 0; g < L->ngauss[f]; ++g) afM *= af;", "afM = af;",
     P2, "test_df_cell_product_mixed_gauss_points", {}),
    ("df_min_not_product", C, "if (alpha) alpha[l] *= afM;", "if (alpha) alpha[l] = fmin(alpha[l], afM);",
     P2, "test_df_cell_product_mixed_gauss_points", {}),
    ("df_Mat_not_squared", C, "dMt2 += t * t;", "dMt2 += fabs(t);", P2, "test_df_tangential_mach_term", {}),
    ("df_Mat_magnitudes", C, "double t = (ul[k] - Ul * n[k]) / al - (ur[k] - Ur * n[k]) / ar;",
     "double t = fabs(ul[k] - Ul * n[k]) / al - fabs(ur[k] - Ur * n[k]) / ar;", P2, "test_df_tangential_mach_term",
     {}),
    ("df_Man_dropped", C, "double D = fabs(pl - pr) / pl + fabs(pl - pr) / pr + dMn * dMn + dMt2;",
     "double D = fabs(pl - pr) / pl + fabs(pl - pr) / pr + dMt2;", P1, "test_df_examples", {}),
    # spectral radius / Sigma (A5, A6)
    ("sigma_interior_only", C, "if (Sigma) Sigma[l] += S * rr;", "if (Sigma && r >= 0) Sigma[l] += S * rr;",
     P2, "test_sigma_single_boundary_cell_hand_computed", {}),
    ("r_of_left_state_only", C, "Wb[q] = 0.5 * (WL[q] + WR[q]);", "Wb[q] = WL[q];",
     P2, "test_sigma_single_boundary_cell_hand_computed", {}),
    ("slip_ghost_half_reflection", C, "Wg[1 + k] = Wi[1 + k] - 2.0 * mn * n[k];", "Wg[1 + k] = Wi[1 + k] - mn * n[k];",
     P2, "test_sigma_single_boundary_cell_hand_computed", {}),
    # MC-SGS sweep (A1, A7)
    ("sweep_r_sign", C, "sum[q] += S * (T1[q] - T0[q] - rf[f] * dWj[q]);",
     "sum[q] += S * (T1[q] - T0[q] + rf[f] * dWj[q]);", P2, "test_linear_flux_sweep_is_symmetric_gauss_seidel",
     {"mk": "tri"}),
    ("sweep_half_dropped", C, "-(Rt[q * n + i] + 0.5 * alpha[i] * sum[q]) / D[i]",
     "-(Rt[q * n + i] + alpha[i] * sum[q]) / D[i]", P2, "test_linear_flux_sweep_is_symmetric_gauss_seidel",
     {"mk": "box"}),
    ("sweep_backward_runs_forward", C, "int c = half == 0 ? cc + 1 : ncolor - cc;", "int c = cc + 1;",
     P2, "test_linear_flux_sweep_is_symmetric_gauss_seidel", {"mk": "tri"}),
    ("sweep_normal_not_flipped", C, "nn[k] = sigma * A[k] / S;", "nn[k] = A[k] / S;",
     P2, "test_linear_flux_sweep_is_symmetric_gauss_seidel", {"mk": "tri"}),
    ("diag_cfl_swapped", C, "(1.0 - alpha[i]) * (Sigma[i] / cfl_exp)", "(1.0 - alpha[i]) * (Sigma[i] / cfl_imp)",
     P1, "test_hybrid_diagonal_examples", {}),
    # residual / KFVS (O4)
    ("residual_right_sign", C, "for (int q = 0; q < nv; ++q) R[q * n + r] -= S * fF[q * nf + f];",
     "for (int q = 0; q < nv; ++q) R[q * n + r] += S * fF[q * nf + f];", P1, "test_freestream_residual_zero",
     {"mk": 1}),
    ("kfvs_recurrence_coeff", C, "double m3 = U * m2 + (2.0 / (2.0 * lambda)) * m1;",
     "double m3 = U * m2 + (1.0 / (2.0 * lambda)) * m1;", P1, "test_kfvs_equal_states_give_euler_flux",
     {"dim": 3}),
    # explicit step, restriction, prolongation (A9, A13, A15)
    ("explicit_V_over_dt", C, "W[q * n + i] - (cfl_exp / Sigma[i]) * R[q * n + i]",
     "W[q * n + i] - (Sigma[i] / cfl_exp) * R[q * n + i]", P2, "test_explicit_step_worked_example", {}),
    ("restrict_alpha_max", C, "if (af[i] < ac[c]) ac[c] = af[i];", "if (af[i] > ac[c]) ac[c] = af[i];",
     P1, "test_restrict_worked_example", {}),
    ("prolong_sign", C, "Wf[q * nfine + i] + alpha_f[i] * (Wc[q * nc + c] - W0c[q * nc + c])",
     "Wf[q * nfine + i] - alpha_f[i] * (Wc[q * nc + c] - W0c[q * nc + c])", P1,
     "test_restrict_conservation_and_prolong_limits", {}),
    # setup (Algorithms 1 and 3)
    ("hash_product_dropped", C, "return (23u * (l + r) + l * r) % nf_interior;",
     "return (23u * (l + r)) % nf_interior;", P1, "test_face_hash_worked_examples", {}),
    ("color_start_2", C, "color[next_start] = 1;                               /* color(v0) = 1 */",
     "color[next_start] = 2;", P1, "test_coloring_valid_and_matches_brute_force", {"mk": 1}),
    # NEXT-1 oracle (cgks3.c, readings C1-C14)
    ("gks_moment_recurrence", C3, "M[k + 2] = U * M[k + 1] + (double)(k + 1) / (2.0 * lambda) * M[k];",
     "M[k + 2] = U * M[k + 1] + (double)(k) / (2.0 * lambda) * M[k];", P3,
     "test_gks_local_matches_bruteforce_quadrature", {"dim": 3, "seed": 0}),
    ("gks_half_range_sign", C3, "gauss_moments(U, lam, l0, U * l0 - e, g->Mu[2]);",
     "gauss_moments(U, lam, l0, U * l0 + e, g->Mu[2]);", P3, "test_gks_local_matches_bruteforce_quadrature",
     {"dim": 2, "seed": 1}),
    ("gks_time_derivative_sign", C3, "for (int q = 0; q < dim + 2; ++q) b[q] = -b[q];", "", P3,
     "test_gks_local_matches_bruteforce_quadrature", {"dim": 3, "seed": 1}),
    ("gks_internal_dof", C3, "return dim == 3 ? (5.0 - 3.0 * gamma) / (gamma - 1.0)",
     "return dim == 3 ? (3.0 - gamma) / (gamma - 1.0)", P3, "test_gks_free_stream_is_euler_flux", {"dim": 3}),
    ("p2_constraint_offset_dropped", C3, "Cm[r * nk + d + k] = (m2_at(M, j, A, B) + dl[A] * dl[B]) - m2_at(M, i, A, B);",
     "Cm[r * nk + d + k] = m2_at(M, j, A, B) - m2_at(M, i, A, B);", P3, "test_p2_exact_for_quadratic_fields", {"k": 0}),
    ("weno_combination_uncorrected", C3, "double cq = w0 / g0, cl = w1 - w0 * g1 / g0;", "double cq = w0 / g0, cl = w1;",
     P3, "test_weno_combination_consistent_for_linear_data", {"gam0": 0.95}),
    ("cgks3_residual_right_sign", C3, "R[(int64_t)q * n + r] -= S * Fs[q] / dtf;",
     "R[(int64_t)q * n + r] += S * Fs[q] / dtf;", P3, "test_residual_discrete_conservation", {"k": 2}),
]
_RUNNER = textwrap.dedent("""
    import sys
    tmp, root, module, name, params = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4], eval(sys.argv[5])
    sys.path.insert(0, tmp)
    sys.path.insert(1, root)
    import oracle
    assert oracle.__file__.startswith(tmp), oracle.__file__
    oracle.lib()
    import importlib
    mod = importlib.import_module("tests." + module)
    fn = getattr(mod, name)
    kw = dict(params)
    names = fn.__code__.co_varnames[:fn.__code__.co_argcount]
    if "steady" in names:
        kw["steady"] = mod._steady_naca(oracle)
    try:
        if names and names[0] in ("orc", "oracle"):
            fn(oracle, **kw)
        else:                # the NEXT-1 pins import oracle.cgks3 themselves (the mutant copy: first on sys.path)
            fn(**kw)
    except AssertionError:
        sys.exit(3)          # the pin fails on the mutant: killed
    sys.exit(0)              # survived
""")


def _mutant_dir(tmp_path, fname, old, new):
    d = tmp_path / "oracle"
    d.mkdir()
    src = os.path.join(ROOT, "oracle")
    for f in os.listdir(src):
        if f.endswith((".c", ".py")):
            shutil.copy(os.path.join(src, f), d / f)
    text = (d / fname).read_text()
    # every occurrence (F appears in both the KFVS and the CGKS3 V-cycle orchestration)
    assert text.count(old) >= 1, f"mutation site absent: {old!r}"
    (d / fname).write_text(text.replace(old, new))
    return str(tmp_path)


@pytest.mark.parametrize("mid,fname,old,new,module,name,params", MUTANTS, ids=[m[0] for m in MUTANTS])
def test_pin_kills_mutant(tmp_path, mid, fname, old, new, module, name, params):
    tmp = _mutant_dir(tmp_path, fname, old, new)
    r = subprocess.run([sys.executable, "-c", _RUNNER, tmp, ROOT, module, name, repr(params)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 3, f"mutant {mid} survived {module}.{name} (rc {r.returncode})\n{r.stdout}\n{r.stderr}"
