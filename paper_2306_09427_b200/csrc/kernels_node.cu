// Node-centric resident DR kernel instances (dr_node.cuh), by preference: an entry takes the
// first shape whose node slots and shared-memory footprint hold it.  MINB is the CTAs per
// SM the register budget is sized for.
#include "variants.hpp"

namespace fibra_b200 {

#define FB_NL(T, N, L, B) {&dr_node_kernel<T, N, L, B, false>, &dr_node_kernel<T, N, L, B, true>}
#define FB_NV(T, N, B) \
  {T, N, B, {FB_NL(T, N, 0, B), FB_NL(T, N, 1, B), FB_NL(T, N, 2, B), FB_NL(T, N, 3, B)}}
const NodeVariant kNodeVariants[] = {
    FB_NV(256, 1, 3),   // <= 256 node slots
    FB_NV(384, 1, 3),   // <= 384 node slots (config 1/2 networks: 375 nodes)
    FB_NV(384, 1, 2),   // the same at 2 CTAs per SM (FIBRA_NODE_SHAPE=2: timing A/B)
    FB_NV(512, 1, 2),   // <= 512 node slots
    FB_NV(512, 2, 1),   // <= 1024 node slots
};
#undef FB_NV
#undef FB_NL
const int kNumNodeVariants = sizeof(kNodeVariants) / sizeof(kNodeVariants[0]);

}  // namespace fibra_b200
