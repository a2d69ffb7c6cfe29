// HBM-streaming DR kernel instances (dr_stream.cuh), per-CTA shapes; an entry too large for
// every resident shape and every cluster shape takes the smallest cluster (C = 2..16) of the
// first shape whose C*T*NPT node slots hold it.
#include "variants.hpp"

namespace fibra_b200 {

#define FB_SL(T, N, L) {&dr_stream_kernel<T, N, L, false>, &dr_stream_kernel<T, N, L, true>}
#define FB_SV(T, N) {T, N, {FB_SL(T, N, 0), FB_SL(T, N, 1), FB_SL(T, N, 2), FB_SL(T, N, 3)}}
const StreamVariant kStreamVariants[] = {
    FB_SV(512, 1),  // <= 8,192 nodes on 16 CTAs
    FB_SV(512, 2),  // <= 16,384 nodes
    FB_SV(512, 4),  // <= 32,768 nodes (~130k fibres)
};
#undef FB_SV
#undef FB_SL
const int kNumStreamVariants = sizeof(kStreamVariants) / sizeof(kStreamVariants[0]);

}  // namespace fibra_b200
