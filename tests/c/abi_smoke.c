/* Plain-C client of the C ABI (include/permkit_b200.h): links
 * libpk_b200.so, checks the version, and walks a 12 x 12 matrix when a
 * device is present (else expects the loud PK_ERR_CUDA, never a CPU result).
 * Built and run by tests/test_c_abi.py. */
#include <stdio.h>
#include <stdlib.h>

#include "permkit_b200.h"

int main(void) {
  if (pk_abi_version() != PK_ABI_VERSION) return 10;
  const int n = 12;
  double a[12 * 12], cols[11 * 12], x0[12], out[2];
  unsigned s = 12345u;
  for (int k = 0; k < n * n; ++k) {
    s = s * 1103515245u + 12345u;
    a[k] = (double)(s >> 8) / 16777216.0;
  }
  for (int j = 0; j < n - 1; ++j)
    for (int i = 0; i < n; ++i) cols[j * n + i] = a[i * n + j];
  for (int i = 0; i < n; ++i) {
    double r = a[i * n];
    for (int j = 1; j < n; ++j) r += a[i * n + j];
    x0[i] = a[i * n + n - 1] - r / 2.0;
  }
  pk_run_stats st;
  const int rc = pk_dense_f64(cols, x0, n, 1, (1ull << (n - 1)) - 1, PK_POLICY_KAHAN, 0, 0, NULL,
                              0, out, &st);
  const int ndev = pk_device_count();
  if (ndev <= 0) {
    /* no device: a loud CUDA error with a message, no CPU fallback */
    if (rc != PK_ERR_CUDA || pk_last_error()[0] == 0) return 11;
    printf("no-device rc=%d msg=%s\n", rc, pk_last_error());
    return 0;
  }
  if (rc != PK_OK) {
    fprintf(stderr, "%s\n", pk_last_error());
    return 12;
  }
  double p0 = 1.0;
  for (int i = 0; i < n; ++i) p0 *= x0[i];
  printf("perm=%.17g updates=%llu launches=%d\n", (p0 + out[0] + out[1]) * (n % 2 ? 2.0 : -2.0),
         (unsigned long long)st.iterates, st.launches);
  /* argument errors map to PK_ERR_ARG (ValueError) */
  if (pk_dense_f64(cols, x0, n, 0, 5, PK_POLICY_KAHAN, 0, 0, NULL, 0, out, NULL) != PK_ERR_ARG)
    return 13;
  return 0;
}
