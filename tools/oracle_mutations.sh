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
  if timeout 600 python -m pytest tests/test_oracle_material.py tests/test_oracle_assembly.py -q -x -m "not slow" >/dev/null 2>&1; then
    echo "NOT CAUGHT: $1 -> $2"; fail=1
  else
    echo "caught:     $1 -> $2"
  fi
}
mut "0.25 * Jd * Ci" "0.26 * Jd * Ci"
mut "double s = (i == kk) ? S[J * 3 + L] : 0.0;" "double s = 0.0;"
mut "f2 * dy[j * 3 + p] * dy[j * 3 + q]" "f2 * dy[j * 3 + p] * dy[j * 3 + p]"
mut "h[1][I * 3 + J] = I1 * d - C[I * 3 + J];" "h[1][I * 3 + J] = I1 * d - C[J * 3 + I] * 1.0000001;"
mut "H[8] += 2.0 * m->kappa;" "H[8] += 1.0 * m->kappa;"
mut "s += F[i * 3 + I] * CC[I4(I, J, K, L)] * F[kk * 3 + K];" "s += F[i * 3 + I] * CC[I4(I, J, K, L)] * F[K * 3 + kk];"
mut "if (B) t += B[j * 3 + p];" ""
mut "F[i * 3 + J] += u[3 * node + i] * gN[a * 3 + J];" "F[i * 3 + J] += u[3 * node + J] * gN[a * 3 + i];"
mut "r[3 * (node - node_begin) + i] += wq * s;" "r[3 * (node - node_begin) + i] += s;"
mut "double I2 = 0.5 * (I1 * I1 - trC2);" "double I2 = 0.5 * (I1 * I1 + trC2);"
exit $fail
