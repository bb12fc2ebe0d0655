#!/usr/bin/env bash
# Mutation check of the oracle pins: each line plants one plausible mistake
# in oracle/oracle.c (wrong coefficient, dropped term, transposed index) and
# requires the CPU pin suite to fail. Restores the original at the end.
set -u
cd "$(dirname "$0")/.."
cp oracle/oracle.c /tmp/oracle_orig.c
trap 'cp /tmp/oracle_orig.c oracle/oracle.c; python -c "import oracle; oracle.build(force=True)"' EXIT
fail=0
mut() {
  cp /tmp/oracle_orig.c oracle/oracle.c
  python - "$1" "$2" <<'PY'
import sys
p = 'oracle/oracle.c'; s = open(p).read(); a, b = sys.argv[1], sys.argv[2]
assert a in s, a
open(p, 'w').write(s.replace(a, b, 1))
PY
  if timeout 600 python -m pytest tests/test_oracle_material.py tests/test_oracle_assembly.py \
      tests/test_oracle_variants.py tests/test_oracle_newton.py -q -x -m "not slow" >/dev/null 2>&1; then
    echo "NOT CAUGHT: $1 -> $2"; fail=1
  else
    echo "caught:     $1 -> $2"
  fi
}
mut "0.25 * Jd * Ci" "0.26 * Jd * Ci"
mut "double s = (i == kk) ? S[J * 3 + L] : 0.0;" "double s = 0.0;"
mut "f2 * dy[j * nk + p] * dy[j * nk + q]" "f2 * dy[j * nk + p] * dy[j * nk + p]"
mut "h[1][I * 3 + J] = I1 * d - C[I * 3 + J];" "h[1][I * 3 + J] = I1 * d - C[J * 3 + I] * 1.0000001;"
mut "H[8] += 2.0 * m->kappa;" "H[8] += 1.0 * m->kappa;"
mut "s += F[i * 3 + I] * CC[I4(I, J, K, L)] * F[kk * 3 + K];" "s += F[i * 3 + I] * CC[I4(I, J, K, L)] * F[K * 3 + kk];"
mut "if (B) t += B[j * 3 + p];" ""
mut "F[i * 3 + J] += u[3 * node + i] * gN[a * 3 + J];" "F[i * 3 + J] += u[3 * node + J] * gN[a * 3 + i];"
mut "r[3 * (node - node_begin) + i] += wq * s;" "r[3 * (node - node_begin) + i] += s;"
mut "double I2 = 0.5 * (I1 * I1 - trC2);" "double I2 = 0.5 * (I1 * I1 + trC2);"
# the ICNN on 5 (anisotropic) inputs: W1 is [w][nk]
mut "for (int i = 0; i < nin; i++) s += A[(size_t)j * nin + i] * z[i];" "for (int i = 0; i < nin; i++) s += A[(size_t)j * (k == 1 ? 3 : nin) + i] * z[i];"
# the s8(f) variants: isochoric G-tensor table, CANN chain rule, Gent-Thomas
mut "const double Ib[2] = {Ib1, Ib2}, e[2] = {-1.0 / 3.0, -2.0 / 3.0};" "const double Ib[2] = {Ib1, Ib2}, e[2] = {-1.0 / 3.0, -1.0 / 3.0};"
mut "GGb[1][I4(i, j, k, l)] = Bb[i * 3 + j] * Bb[k * 3 + l] -" "GGb[1][I4(i, j, k, l)] = Bb[i * 3 + j] * Bb[k * 3 + l] +"
mut "e[mm] * ((i == j) * Gb[mm][k * 3 + l] + Gb[mm][i * 3 + j] * (k == l)" "e[mm] * ((i == j) * Gb[mm][k * 3 + l]"
mut "t += Fi[I * 3 + i] * Fi[J * 3 + j] * Fi[K * 3 + k] * Fi[L * 3 + l] * c[I4(i, j, k, l)];" "t += Fi[I * 3 + i] * Fi[J * 3 + j] * Fi[K * 3 + l] * Fi[L * 3 + k] * c[I4(i, j, k, l)] * 1.0000001;"
mut "dd2 = w1 * w1 / ((1.0 - w1 * v1) * (1.0 - w1 * v1));" "dd2 = -w1 * w1 / ((1.0 - w1 * v1) * (1.0 - w1 * v1));"
mut "H[mm * nin + mm] += w2 * ((dd2 * d1 * d1 + d2 * dd1) * d0 * d0" "H[mm * nin + mm] += w2 * ((dd2 * d1 + d2 * dd1) * d0 * d0"
mut "H[4] = -m->gt[1] / ((K[1] + 3.0) * (K[1] + 3.0));" "H[4] = m->gt[1] / ((K[1] + 3.0) * (K[1] + 3.0));"
# ICKAN: De Boor recursion and spline derivatives
mut "if (t[i + p + 1] > t[i + 1]) v += (t[i + p + 1] - x) / (t[i + p + 1] - t[i + 1]) * B[(p - 1) * nt + i + 1];" "if (t[i + p + 1] > t[i + 1]) v += (t[i + p + 1] - x) / (t[i + p + 1] - t[i]) * B[(p - 1) * nt + i + 1];"
mut "for (int q = 0; q < nk; q++) d2y[i][p * nk + q] += w * (d2 * dz[j][p] * dz[j][q] + d1 * d2z[j][p * nk + q]);" "for (int q = 0; q < nk; q++) d2y[i][p * nk + q] += w * (d2 * dz[j][p] * dz[j][q]);"
# anisotropic I4,ij / I5,ij (the paper's G-tensor table, several structural vectors)
mut "G[m5][i * 3 + j] = 0.5 * (ai[i] * Baj[j] + Baj[i] * ai[j]) + 0.5 * (aj[i] * Bai[j] + Bai[i] * aj[j]);" "G[m5][i * 3 + j] = 0.5 * (ai[i] * Baj[j] + Baj[i] * ai[j]) + 0.5 * (aj[i] * Bai[j] + B[i * 3 + j]);"
mut "GG[m5][x] = 0.5 * (B[i * 3 + k] * As[j * 3 + l] + B[i * 3 + l] * As[j * 3 + k]) +" "GG[m5][x] = 0.5 * (B[i * 3 + k] * As[j * 3 + l] + B[i * 3 + l] * As[j * 3 + k]) * 0.0 +"
# reading R28: the table's literal G^{5,ij} = 2 sym(a_i (x) B a_j) for i != j
mut "G[m5][i * 3 + j] = 0.5 * (ai[i] * Baj[j] + Baj[i] * ai[j]) + 0.5 * (aj[i] * Bai[j] + Bai[i] * aj[j]);" "G[m5][i * 3 + j] = (ai[i] * Baj[j] + Baj[i] * ai[j]);"
mut "i4 += Ai[I] * CAj[I];   /* A_i.C A_j */" "i4 += Ai[I] * CAi[I];   /* A_i.C A_j */"
mut "G[m4][i * 3 + j] = As[i * 3 + j];" "G[m4][i * 3 + j] = ai[i] * aj[j];"
# isochoric anisotropic (App. A.2.2 with Ibar4,ij / Ibar5,ij; reading R29)
mut "kN[4 + 2 * p] = a23 * a23 * i5 - aa;" "kN[4 + 2 * p] = a23 * i5 - aa;"
mut "    e[m5] = -2.0 / 3.0;" "    e[m5] = -1.0 / 3.0;"
mut "Bab[v][i] = Bb[i * 3] * ab[v][0] + Bb[i * 3 + 1] * ab[v][1] + Bb[i * 3 + 2] * ab[v][2];" "Bab[v][i] = (Bb[i * 3] * ab[v][0] + Bb[i * 3 + 1] * ab[v][1] + Bb[i * 3 + 2] * ab[v][2]) / (c13 * c13);"
mut "GGb[m5][x] = 0.5 * (Bb[i * 3 + k] * As[j * 3 + l] + Bb[i * 3 + l] * As[j * 3 + k]) +" "GGb[m5][x] = 0.5 * (Bb[i * 3 + k] * As[j * 3 + l] + Bb[i * 3 + l] * As[j * 3 + k]) * 0.0 +"
mut "Gb[m4][i * 3 + j] = As[i * 3 + j];" "Gb[m4][i * 3 + j] = ai[i] * aj[j];"
mut "    if (mm == 2) continue;" "    if (mm == 2 || mm >= 3) continue;"
exit $fail
