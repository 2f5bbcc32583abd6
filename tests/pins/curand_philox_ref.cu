// Pin P1 (tests only): NVIDIA cuRAND's own Philox4x32-10 (curand_philox4x32_x.h,
// host path of mulhilo32) evaluated on the host -- an implementation independent
// of both oracle/asaga_oracle.c and the CUDA product path.
#include <stdint.h>
#include <vector_types.h>
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>

extern "C" void curand_ref_philox_stream(uint64_t seed, uint64_t t0, uint64_t count,
                                         uint32_t* out) {
  for (uint64_t k = 0; k < count; ++k) {
    uint64_t t = t0 + k;
    uint4 c = make_uint4((unsigned)t, (unsigned)(t >> 32), 0u, 0u);
    uint2 key = make_uint2((unsigned)seed, (unsigned)(seed >> 32));
    uint4 r = curand_Philox4x32_10(c, key);
    out[4 * k + 0] = r.x; out[4 * k + 1] = r.y; out[4 * k + 2] = r.z; out[4 * k + 3] = r.w;
  }
}
