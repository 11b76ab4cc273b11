// Seeded synthetic inputs for the BASELINE configs (host side, not on the hot path).
// Engine and uniform draw follow the reference's Rng (include/cloth/rng.hpp:12-46):
// std::mt19937_64, uniform01 = (u64 >> 11) * 2^-53, independent streams via Rng::mix
// (splitmix64 finaliser, rng.hpp:36-42). Normals: Box-Muller over uniform01, both outputs used
// (this repo's frozen convention). Per-(cloth, row) noise streams make every
// cloth's and every row's inputs independent of how work is partitioned across GPUs.
#include <cmath>
#include <cstdint>
#include <random>
#include <thread>
#include <vector>

namespace {

uint64_t mix(uint64_t seed, uint64_t stream) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

struct Gen {
  std::mt19937_64 g;
  bool have = false;
  double spare = 0.0;
  explicit Gen(uint64_t s) : g(s) {}
  double u01() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
  double normal() {
    if (have) {
      have = false;
      return spare;
    }
    const double u1 = u01(), u2 = u01();
    const double r = std::sqrt(-2.0 * std::log(1.0 - u1));
    const double a = 6.283185307179586476925286766559 * u2;
    spare = r * std::sin(a);
    have = true;
    return r * std::cos(a);
  }
};

}  // namespace

extern "C" {

uint64_t sc_rng_mix(uint64_t seed, uint64_t stream) { return mix(seed, stream); }

// the first `count` raw outputs of std::mt19937_64(seed): the engine under cloth::Rng
// (rng.hpp:13-47), whose fixed-algorithm draws the Python layer builds on
void sc_mt64_fill(uint64_t seed, int64_t count, uint64_t* out) {
  std::mt19937_64 g(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = g();
}

// count uniforms in [0,1) from one stream
void sc_rng_uniform01(uint64_t seed, int64_t count, double* out) {
  Gen g(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = g.u01();
}

// count normals N(0, sigma^2) from one stream
void sc_rng_normal(uint64_t seed, int64_t count, double sigma, double* out) {
  Gen g(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = sigma * g.normal();
}

// Flat nx-by-ny sheet (build_grid(nx, ny, spacing, origin, XY), reference grid.cpp:118-135)
// plus N(0, sigma^2) noise on all three components; row iy of cloth `cloth` draws from stream
// mix(mix(seed, 0x10000 + cloth), iy). Rows [row0, row0 + rows) only (strip shards).
// out_f32 / out_f64: AoS [rows][nx][3] (either may be null).
void sc_gen_sheet(uint64_t seed, int64_t cloth, int32_t nx, int32_t ny, int32_t row0,
                  int32_t rows, double spacing, double sigma, float* out_f32, double* out_f64,
                  int32_t threads) {
  (void)ny;
  const uint64_t cs = mix(seed, 0x10000ULL + static_cast<uint64_t>(cloth));
  auto work = [&](int r_begin, int r_end) {
    for (int r = r_begin; r < r_end; ++r) {
      const int iy = row0 + r;
      Gen g(mix(cs, static_cast<uint64_t>(iy)));
      for (int ix = 0; ix < nx; ++ix) {
        const double base[3] = {spacing * ix, spacing * iy, 0.0};
        for (int d = 0; d < 3; ++d) {
          const double v = base[d] + sigma * g.normal();
          const int64_t o = (static_cast<int64_t>(r) * nx + ix) * 3 + d;
          if (out_f32) out_f32[o] = static_cast<float>(v);
          if (out_f64) out_f64[o] = v;
        }
      }
    }
  };
  if (threads <= 1 || rows < 64) {
    work(0, rows);
    return;
  }
  std::vector<std::thread> pool;
  const int per = (rows + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const int b = t * per, e = std::min(rows, b + per);
    if (b < e) pool.emplace_back(work, b, e);
  }
  for (auto& t : pool) t.join();
}

}  // extern "C"
