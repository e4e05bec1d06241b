// Library pin for the oracle's Philox4x32-10 (tests/test_oracle_philox.py):
// cuRAND's own Philox round function, compiled for the HOST from the CUDA
// toolkit header (QUALIFIERS predefined so the header's functions are host
// callable).  This is NOT part of the oracle or of the product path.
#include <cstdint>
#include <vector_types.h>
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>

extern "C" void pin_curand_philox(uint64_t seed, const uint32_t* ctr, int64_t n, uint32_t* out) {
  uint2 key; key.x = (uint32_t)seed; key.y = (uint32_t)(seed >> 32);
  for (int64_t i = 0; i < n; ++i) {
    uint4 c; c.x = ctr[4*i]; c.y = ctr[4*i+1]; c.z = ctr[4*i+2]; c.w = ctr[4*i+3];
    uint4 r = curand_Philox4x32_10(c, key);
    out[4*i] = r.x; out[4*i+1] = r.y; out[4*i+2] = r.z; out[4*i+3] = r.w;
  }
}
