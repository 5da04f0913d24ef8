"""Mutation check of the oracle's pins: apply one plausible mistake at a time to a copy of
oracle/ (a dropped term, a wrong sign or index, a transposed operand, a mis-scaled metric),
rebuild it, run tests/test_oracle_pins.py, and report every mutation the pins did NOT catch.

    python tools/oracle_mutations.py            # CPU only, a few minutes
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (file, original text, mutated text, description); each original must occur exactly once
MUTATIONS = [
    # CRIT (upper), Alg. 3
    ("oracle.c", "for (int64_t k = i; k < j; ++k) dot += AT(S, lds, i, k) * AT(R, ldr, k, j);",
     "for (int64_t k = i + 1; k < j; ++k) dot += AT(S, lds, i, k) * AT(R, ldr, k, j);", "crit_upper: k-range drops k = i"),
    ("oracle.c", "AT(S, lds, i, j) = unit ? -dot : -dot / AT(R, ldr, j, j);",
     "AT(S, lds, i, j) = unit ? -dot : -dot / AT(R, ldr, i, i);", "crit_upper: divides by R_ii"),
    ("oracle.c", "for (int64_t k = i; k < j; ++k) dot += AT(S, lds, i, k) * AT(R, ldr, k, j);",
     "for (int64_t k = i; k < j; ++k) dot += AT(S, lds, i, k) * AT(R, ldr, j, k);", "crit_upper: R transposed"),
    ("oracle.c", "AT(S, lds, i, j) = unit ? -dot : -dot / AT(R, ldr, j, j);",
     "AT(S, lds, i, j) = unit ? dot : -dot / AT(R, ldr, j, j);", "crit_upper: unit sign"),
    ("oracle.c", "AT(S, lds, i, i) = unit ? 1.0 : 1.0 / AT(R, ldr, i, i);",
     "AT(S, lds, i, i) = unit ? AT(R, ldr, i, i) : 1.0 / AT(R, ldr, i, i);", "crit_upper: unit reads the diagonal"),
    # lower (transpose)
    ("oracle.c", "for (int64_t k = i; k < j; ++k) dot += AT(X, ldx, k, i) * AT(L, ldl, j, k);",
     "for (int64_t k = i; k < j - 1; ++k) dot += AT(X, ldx, k, i) * AT(L, ldl, j, k);", "crit_lower: drops k = j-1"),
    ("oracle.c", "AT(X, ldx, j, i) = unit ? -dot : -dot / AT(L, ldl, j, j);",
     "AT(X, ldx, j, i) = unit ? -dot : dot / AT(L, ldl, j, j);", "crit_lower: sign"),
    ("oracle.c", "for (int64_t k = i; k < j; ++k) dot += AT(X, ldx, k, i) * AT(L, ldl, j, k);",
     "for (int64_t k = i; k < j; ++k) dot += AT(X, ldx, k, i) * AT(L, ldl, k, j);", "crit_lower: L transposed"),
    ("oracle.c", "for (int64_t j = 0; j < i; ++j) AT(X, ldx, j, i) = 0.0;",
     "for (int64_t j = 0; j + 1 < i; ++j) AT(X, ldx, j, i) = 0.0;", "crit_lower: one structural zero left unwritten"),
    # batched lower
    ("oracle.c", "for (int64_t k = i; k < j; ++k) dot += AT(Y, ldx, k, i) * AT(L, lda, j, k);",
     "for (int64_t k = i + 1; k < j; ++k) dot += AT(Y, ldx, k, i) * AT(L, lda, j, k);", "batched: drops k = i"),
    ("oracle.c", "AT(Y, ldx, j, i) = unit ? -dot : -dot / AT(L, lda, j, j);",
     "AT(Y, ldx, j, i) = unit ? -dot : -dot / AT(L, lda, i, i);", "batched: divides by L_ii"),
    ("oracle.c", "    oracle_crit_upper(n, A + b * sA, lda, X + b * sX, ldx, unit);",
     "    oracle_crit_upper(n, A + b * sA, lda, X + b * sX, ldx, 0);", "batched upper: unit flag dropped"),
    # sampled columns
    ("oracle.c", "for (int64_t k = j; k < i; ++k) dot += x[k] * AT(L, ldl, i, k);",
     "for (int64_t k = j + 1; k < i; ++k) dot += x[k] * AT(L, ldl, i, k);", "lower_column: drops k = j"),
    ("oracle.c", "x[i] = unit ? -dot : -dot / AT(L, ldl, i, i);",
     "x[i] = unit ? -dot : -dot / AT(L, ldl, j, j);", "lower_column: divides by L_jj"),
    ("oracle.c", "for (int64_t k = i + 1; k <= j; ++k) dot += AT(U, ldu, i, k) * x[k];",
     "for (int64_t k = i + 1; k < j; ++k) dot += AT(U, ldu, i, k) * x[k];", "upper_column: drops k = j"),
    ("oracle.c", "x[i] = unit ? -dot : -dot / AT(U, ldu, i, i);",
     "x[i] = unit ? -dot : -dot / AT(U, ldu, j, j);", "upper_column: divides by U_jj"),
    ("oracle.c", "    else oracle_upper_column(n, T, ld, unit, cols[c], out + c * n);",
     "    else oracle_upper_column(n, T, ld, unit, cols[c] > 0 ? cols[c] - 1 : 0, out + c * n);", "columns: off-by-one column"),
    # inv_from_lu columns
    ("oracle.c", "    for (int64_t k = i + 1; k < n; ++k) s -= AT(U, ldu, i, k) * x[k];",
     "    for (int64_t k = i + 1; k < n; ++k) s += AT(U, ldu, i, k) * x[k];", "lu_column: sign of the U update"),
    ("oracle.c", "    x[i] = unitU ? s : s / AT(U, ldu, i, i);",
     "    x[i] = s / AT(U, ldu, i, i) * (unitU ? AT(U, ldu, i, i) : 1.0) + 0.0 * unitU;", "lu_column: (no-op rewrite, must survive)"),
    ("oracle.c", "    for (int64_t k = i + 1; k < n; ++k) s -= AT(U, ldu, i, k) * x[k];",
     "    for (int64_t k = i + 1; k < n; ++k) s -= AT(U, ldu, k, i) * x[k];", "lu_column: U transposed"),
    # path sum (Thm 1)
    ("oracle.c", "          s += ((len - 1) % 2) ? -prod : prod; /* (-1)^(l-1) */",
     "          s += (len % 2) ? -prod : prod; /* (-1)^(l-1) */", "pathsum: sign convention"),
    ("oracle.c", "              double Tab = unit ? AT(R, ldr, a, nxt) : AT(R, ldr, a, nxt) / AT(R, ldr, a, a);",
     "              double Tab = unit ? AT(R, ldr, a, nxt) : AT(R, ldr, a, nxt) / AT(R, ldr, nxt, nxt);", "pathsum: scales by the wrong diagonal"),
    ("oracle.c", "      AT(X, ldx, i, j) = unit ? s : s / AT(R, ldr, j, j);",
     "      AT(X, ldx, i, j) = unit ? s : s / AT(R, ldr, i, i);", "pathsum: final division by R_ii"),
    ("oracle.c", "        for (uint64_t mask = 0; mask < (1ULL << m); ++mask) {",
     "        for (uint64_t mask = 0; mask + 1 < (1ULL << m); ++mask) {", "pathsum: drops the full-interior path"),
    # SKUL
    ("oracle.c", "      for (int64_t p = 0; p < j; ++p) dot += L[i * N + p] * U[p * N + j];\n      L[i * N + j] = A[i * N + j] - dot;",
     "      for (int64_t p = 0; p + 1 < j; ++p) dot += L[i * N + p] * U[p * N + j];\n      L[i * N + j] = A[i * N + j] - dot;", "skul: L dot drops a term"),
    ("oracle.c", "      for (int64_t p = 0; p <= i; ++p) dot += L[i * N + p] * K[p * N + j];",
     "      for (int64_t p = 0; p < i; ++p) dot += L[i * N + p] * K[p * N + j];",
     "skul: K dot drops p = i (equivalent: K_ij is still 0 when it is formed, must survive)"),
    ("oracle.c", "K[i * N + j] *= D[j];", "K[i * N + j] *= D[i];", "skul: K D with the wrong index"),
    ("oracle.c", "        S[l * N + i + 1] = -dot;",
     "        S[l * N + i + 1] = dot;", "skul: S sign"),
    ("oracle.c", "      U[i * N + j] = (A[i * N + j] - dot) / L[i * N + i];",
     "      U[i * N + j] = (A[i * N + j] - dot) / L[j * N + j];", "skul: U divides by L_jj"),
    # metrics
    ("metrics.py", "    num = np.sqrt(np.sum(E * E, axis=(-2, -1)))", "    num = np.sum(E * E, axis=(-2, -1))",
     "residual_ratio: sqrt dropped"),
    ("metrics.py", "    return float(np.max(num / den))", "    return float(np.mean(num / den))", "residual_ratio: mean over the batch"),
    ("metrics.py", "    E = T @ X - np.eye(n)", "    E = X @ T - np.eye(n)", "residual_ratio: X T for T X"),
    ("metrics.py", "    E[np.asarray(cols), np.arange(len(cols))] -= 1.0\n    return float(np.linalg.norm(E) / (np.linalg.norm(T) * np.linalg.norm(Xs)))",
     "    E[np.asarray(cols), np.arange(len(cols))] -= 1.0\n    return float(np.linalg.norm(E) / (np.linalg.norm(T) * np.linalg.norm(Xs)) * 0)",
     "column_residual_ratio: constant 0"),
    ("metrics.py", "        colmax = np.max(np.abs(R), axis=-2, keepdims=True)", "        colmax = np.max(np.abs(R), axis=-1, keepdims=True)",
     "floored_rel_err: floor over rows instead of columns"),
    ("metrics.py", "    den = np.maximum(np.abs(R), floor * colmax)", "    den = np.maximum(np.abs(R), colmax)",
     "floored_rel_err: floor factor dropped"),
    ("metrics.py", "    E = L @ (U @ Xs)", "    E = U @ (L @ Xs)", "factored residual: U L for L U"),
    # Python wrappers and the Hopscotch enumerator
    ("__init__.py", "    f = lib().oracle_crit_lower_batched if uplo == \"L\" else lib().oracle_crit_upper_batched",
     "    f = lib().oracle_crit_upper_batched if uplo == \"L\" else lib().oracle_crit_lower_batched",
     "crit_batched: uplo swapped"),
    ("__init__.py", "    lib().oracle_lu_columns(n, _p(L), n, int(unit_l), _p(U), n, int(unit_u), len(cols),",
     "    lib().oracle_lu_columns(n, _p(L), n, int(unit_u), _p(U), n, int(unit_l), len(cols),",
     "lu_columns: unit flags swapped"),
    ("__init__.py", "    return S @ K", "    return K @ S", "inv_general: K S for S K"),
    ("hopscotch.py", "    for k in range(len(interior), -1, -1):", "    for k in range(len(interior), 0, -1):",
     "hopscotch: drops the direct hop a -> b"),
    ("hopscotch.py", "    interior = list(range(a + 1, b))", "    interior = list(range(a + 1, b + 1))",
     "hopscotch: interior includes b"),
]


def main():
    survivors, errors = [], []
    for idx, (fname, old, new, what) in enumerate(MUTATIONS):
        with tempfile.TemporaryDirectory() as tmp:
            for d in ("oracle", "tests", "synth"):
                shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                                ignore=shutil.ignore_patterns("*.so", "__pycache__"))
            for f in ("pytest.ini", "conftest.py", "setup.cfg", "pyproject.toml"):
                if os.path.exists(os.path.join(ROOT, f)):
                    shutil.copy(os.path.join(ROOT, f), tmp)
            path = os.path.join(tmp, "oracle", fname)
            src = open(path).read()
            if src.count(old) != 1:
                errors.append((what, f"pattern occurs {src.count(old)} times"))
                continue
            open(path, "w").write(src.replace(old, new))
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                                "tests/test_oracle_pins.py"], cwd=tmp, capture_output=True, text=True, timeout=900)
            caught = r.returncode != 0
            print(f"{idx:2d} {'caught  ' if caught else 'SURVIVED'} {what}", flush=True)
            if not caught:
                survivors.append(what)
    print(f"\n{len(MUTATIONS) - len(errors) - len(survivors)} caught, {len(survivors)} survived, "
          f"{len(errors)} not applied")
    for w in survivors:
        print("  survived:", w)
    for w, e in errors:
        print("  not applied:", w, e)


if __name__ == "__main__":
    main()
