// The fp32 tcgen05 kernel in its CTA-pair form (umma_f32.cu, TC_UMMA_PAIR): clusters of two CTAs,
// tcgen05.mma.cta_group::2 with M = 256 issued by the leader, each CTA staging its 128 rows of A
// and half of B.
#define TC_UMMA_PAIR 1
#define TC_UMMA_NS umma_pair
#define TC_UMMA_LAUNCH launch_umma_f32_pair
#include "umma_f32.cu"
