/* tsgen_host.c — host-side fill of the seeded synthetic potentials (tsgen.h).
 * Exported for the Python generator module (bit-equality test against numpy and
 * against the device fill).  Test/bench infrastructure only. */
#include <stdint.h>

#include "tsgen.h"

int tsgen_fill_host(float* out, int64_t B, int64_t E_local, int64_t C, uint64_t seed, int s,
                    int64_t t_begin, int64_t E_global) {
  if (B <= 0 || E_local <= 0 || C <= 0) return 0;
  if (!out || s < 0 || s > 15 || t_begin < 0 || t_begin + E_local > E_global) return 1;
  int64_t n = 0;
  for (int64_t b = 0; b < B; ++b)
    for (int64_t t = 0; t < E_local; ++t)
      for (int64_t i = 0; i < C; ++i)
        for (int64_t j = 0; j < C; ++j)
          out[n++] = tsgen_value(seed, s, tsgen_index(b, t_begin + t, i, j, E_global, C));
  return 0;
}

int tsgen_quantum_c(int64_t E) { return tsgen_quantum(E); }
