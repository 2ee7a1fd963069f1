/* afem_testing.h — test-only entry points of libafem_b200.so, outside the drop-in boundary
 * (include/afem.h). The slab decomposition's threads backend runs the multi-GPU algorithm with
 * several subdomains on one device (one host thread per subdomain, device copies for the plane
 * exchange and a host barrier for the allreduces) so that the N > 1 data path is exercised where
 * only one GPU exists; production runs use afem_dist_create_nccl. */
#ifndef AFEM_TESTING_H
#define AFEM_TESTING_H

#include "afem.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct afem_thread_group_s* afem_thread_group;

afem_status afem_thread_group_create(int32_t size, afem_thread_group* out);
afem_status afem_thread_group_destroy(afem_thread_group g);
afem_status afem_dist_create_threads(afem_ctx ctx, afem_thread_group g, int32_t rank, afem_dist* out);

#ifdef __cplusplus
}
#endif
#endif /* AFEM_TESTING_H */
