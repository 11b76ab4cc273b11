/*
 * TEST / BENCH INFRASTRUCTURE ONLY — the synthetic BASELINE workloads' inputs, generated on the
 * checker side so bench.py's reference arm and cpu_baseline never load the product library.
 *
 * Restates, in plain C:
 *   std::mt19937_64 (the engine under cloth::Rng, /root/reference/proj/include/cloth/rng.hpp:13-47;
 *     the published MT19937-64 algorithm: n = 312, m = 156, matrix 0xB5026F5AA96619E9,
 *     tempering (29, 0x5555555555555555), (17, 0x71D67FFFEDA60000), (37, 0xFFF7EEE000000000), 43,
 *     initialisation multiplier 6364136223846793005),
 *   Rng::uniform01 (rng.hpp:29: (u64 >> 11) * 2^-53) and Rng::mix (rng.hpp:36-42, the splitmix64
 *     finaliser),
 *   the repo's frozen workload convention: Box-Muller normals (both outputs used),
 *     per-(cloth, row) noise streams mix(mix(seed, 0x10000 + cloth), row), a build_grid sheet
 *     (grid.cpp:118-135) of spacing 1/(n-1) plus N(0, sigma^2) noise on every component.
 * tests/test_workloads.py checks it against the product's generator draw for draw.
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

typedef struct {
  uint64_t mt[312];
  int i;
} orc_mt64;

static void mt64_seed(orc_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->i = 312;
}

static uint64_t mt64_next(orc_mt64* g) {
  static const uint64_t UPPER = 0xFFFFFFFF80000000ULL, LOWER = 0x7FFFFFFFULL;
  if (g->i >= 312) {
    for (int k = 0; k < 312; ++k) {
      const uint64_t x = (g->mt[k] & UPPER) | (g->mt[(k + 1) % 312] & LOWER);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[k] = g->mt[(k + 156) % 312] ^ xa;
    }
    g->i = 0;
  }
  uint64_t y = g->mt[g->i++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

uint64_t orc_rng_mix(uint64_t seed, uint64_t stream) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

typedef struct {
  orc_mt64 g;
  int have;
  double spare;
} orc_gen;

static double gen_u01(orc_gen* s) { return (double)(mt64_next(&s->g) >> 11) * 0x1.0p-53; }

static double gen_normal(orc_gen* s) {
  if (s->have) {
    s->have = 0;
    return s->spare;
  }
  const double u1 = gen_u01(s), u2 = gen_u01(s);
  const double r = sqrt(-2.0 * log(1.0 - u1));
  const double a = 6.283185307179586476925286766559 * u2;
  s->spare = r * sin(a);
  s->have = 1;
  return r * cos(a);
}

void orc_rng_uniform01(uint64_t seed, int64_t count, double* out) {
  orc_gen s;
  mt64_seed(&s.g, seed);
  s.have = 0;
  for (int64_t i = 0; i < count; ++i) out[i] = gen_u01(&s);
}

void orc_rng_normal(uint64_t seed, int64_t count, double sigma, double* out) {
  orc_gen s;
  mt64_seed(&s.g, seed);
  s.have = 0;
  for (int64_t i = 0; i < count; ++i) out[i] = sigma * gen_normal(&s);
}

/* Rows [row0, row0 + rows) of cloth `cloth`'s noisy sheet as AoS [rows][nx][3] floats. */
void orc_gen_sheet(uint64_t seed, int64_t cloth, int32_t nx, int32_t row0, int32_t rows,
                   double spacing, double sigma, float* out) {
  const uint64_t cs = orc_rng_mix(seed, 0x10000ULL + (uint64_t)cloth);
  for (int r = 0; r < rows; ++r) {
    const int iy = row0 + r;
    orc_gen s;
    mt64_seed(&s.g, orc_rng_mix(cs, (uint64_t)iy));
    s.have = 0;
    for (int ix = 0; ix < nx; ++ix) {
      const double base[3] = {spacing * ix, spacing * iy, 0.0};
      for (int d = 0; d < 3; ++d)
        out[((int64_t)r * nx + ix) * 3 + d] = (float)(base[d] + sigma * gen_normal(&s));
    }
  }
}
