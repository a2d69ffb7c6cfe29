// Cluster DR kernel instances (dr_cluster.cuh), per-CTA shapes; an entry that fits no
// resident shape takes the smallest cluster size C = 2, 4, 8, 16 (then the first shape)
// that holds its parts.
#include "variants.hpp"

namespace fibra_b200 {

#define FB_CV(T, F, N)                                                                  \
  {T, F, N,                                                                               \
   {{&dr_cluster_kernel<T, F, N, 0, false>, &dr_cluster_kernel<T, F, N, 0, true>},       \
    {&dr_cluster_kernel<T, F, N, 1, false>, &dr_cluster_kernel<T, F, N, 1, true>}}}
const ClusterVariant kClusterVariants[] = {
    FB_CV(384, 3, 1),  // <= 384 nodes, <= 1056 fibers per CTA (config-3 networks)
    FB_CV(512, 7, 2),  // <= 1024 nodes, <= 3360 fibers per CTA (config-4 networks)
};
#undef FB_CV
const int kNumClusterVariants = sizeof(kClusterVariants) / sizeof(kClusterVariants[0]);

}  // namespace fibra_b200
