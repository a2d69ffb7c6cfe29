// Cluster DR kernel instances (dr_cluster.cuh), per-CTA shapes.  An entry that fits no
// resident shape takes the fewest CTAs (C = 2, 4, 8, 16), then the first shape below that
// holds its parts.
#include "variants.hpp"

namespace fibra_b200 {

#define FB_CL(T, F, N, L) {&dr_cluster_kernel<T, F, N, L, false>, &dr_cluster_kernel<T, F, N, L, true>}
#define FB_CV(T, F, N) \
  {T, F, N, {FB_CL(T, F, N, 0), FB_CL(T, F, N, 1), FB_CL(T, F, N, 2), FB_CL(T, F, N, 3)}}
const ClusterVariant kClusterVariants[] = {
    FB_CV(384, 3, 1),  // <= 384 nodes, <= 1056 fibers per CTA
    FB_CV(384, 4, 1),  // <= 384 nodes, <= 1408 fibers per CTA (config-3 networks)
    FB_CV(512, 7, 2),  // <= 1024 nodes, <= 3360 fibers per CTA (config-4 networks)
};
#undef FB_CV
#undef FB_CL
const int kNumClusterVariants = sizeof(kClusterVariants) / sizeof(kClusterVariants[0]);

}  // namespace fibra_b200
