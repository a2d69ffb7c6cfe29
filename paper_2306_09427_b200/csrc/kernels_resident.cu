// Resident DR kernel instances (dr_kernel.cuh), by preference: an entry takes the first
// shape whose capacity covers it.  MINB = 2 keeps two CTAs (two RVEs) per SM so one CTA's
// barrier wait is covered by the other's work.
#include "variants.hpp"

namespace fibra_b200 {

#define FB_L(T, F, N, L, B) \
  {&dr_persistent_kernel<T, F, N, L, B, false>, &dr_persistent_kernel<T, F, N, L, B, true>}
#define FB_V(T, F, N, B)                                                                 \
  {T, F, N, B,                                                                             \
   {FB_L(T, F, N, 0, B), FB_L(T, F, N, 1, B), FB_L(T, F, N, 2, B), FB_L(T, F, N, 3, B)}}
const Variant kVariants[] = {
    FB_V(256, 3, 1, 2),  // <= 256 node slots, <= 672 fibers
    FB_V(384, 3, 1, 2),  // <= 384 node slots, <= 1056 fibers (config 1/2 networks)
    // (a (512, 2, 1) shape at 2 CTAs/SM held 64 registers and spilled: config 3's 173
    //  points of 385-512 nodes finished 0.5-0.8 s after every other class on it; on
    //  (512, 4, 1) config 3 runs 2,174 -> 2,355 and config 5 1,338 -> 1,553 RVE-solves/s)
    FB_V(512, 4, 1, 1),  // <= 512 node slots, <= 1920 fibers (record offsets in 8-byte units)
    FB_V(512, 6, 2, 1),  // <= 1024 node slots (node-heavy segments networks)
    FB_V(768, 7, 2, 1),  // <= 1536 node slots
};
#undef FB_V
#undef FB_L
const int kNumVariants = sizeof(kVariants) / sizeof(kVariants[0]);

}  // namespace fibra_b200
