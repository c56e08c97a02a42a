// The fp32 tcgen05 kernel in its N = 256 form (umma_f32.cu, TC_UMMA_N256): per K = 8 one
// 128x256 MMA of A hi against [B hi; B lo] and one 128x128 MMA of A lo against B hi, four K steps
// per TMEM chunk. Used when neither operand qualifies for 16-byte vector gathers: there it
// measured faster than the N = 128 form and its accumulation bias is lower (one-signed data:
// -8.5e-7 against -9.6e-7; profiles/r01/ab_umma_n256.txt).
#define TC_UMMA_N256 1
#define TC_UMMA_CHUNK 4
#define TC_UMMA_ELEM_ONLY 1
#define TC_UMMA_NS umma256
#define TC_UMMA_LAUNCH launch_umma_f32_n256
#include "umma_f32.cu"
