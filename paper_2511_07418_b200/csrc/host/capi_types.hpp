// capi_types.hpp — definitions of the host-side opaque C-ABI handles, shared
// by the host translation unit and the device one (lg_hand_patches_device).
#pragma once

#include "host.hpp"

struct lg_hand {
  lgh::Hand h;
};
struct lg_mesh {
  lgh::Mesh m;
  std::vector<double> fv;
  std::vector<int> ft;
};
struct lg_patches {
  lgh::Patches p;
};
