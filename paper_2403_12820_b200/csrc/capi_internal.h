// Internal (non-ABI) hooks between capi.cu and the other host TUs (train.cu): a read-only view
// of an f64 context's device-resident scene constants, and the shared sc_last_error() slot.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/stencilcloth_b200.h"

namespace scb {

struct SceneView {
  const void* cloths;   // ClothConst<T>[batch]
  const void* spheres;  // SphereConst<T>[]
  const void* planes;   // PlaneConst<T>[]
  const void* anchors;  // T[3 * pins]
  const uint32_t* pin_bits;
  const int32_t* pin_rank;
  int nx, ny, batch, device;
};

// false when the context has no scene bound or is a row-strip context
bool ctx_scene_view(sc_ctx* c, SceneView* out);
void set_last_error(const std::string& msg);

}  // namespace scb
