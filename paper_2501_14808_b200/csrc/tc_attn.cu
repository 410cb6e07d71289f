// tc_attn.cu -- tcgen05 / TMEM / TMA flash-attention tiles (prefill chunks and
// shared-prefix group passes).  Placeholder until the kernel lands.
#include "hg_internal.h"

struct hg_kv_pool;
namespace hg {
bool make_tensor_maps(hg_kv_pool *) { return false; }
int tc_supported(int) { return 0; }
hg_status launch_tc(const AttnParams &, const void *, const void *, void *) {
    return fail(HG_E_UNSUPPORTED, "tcgen05 path not built");
}
}  // namespace hg
