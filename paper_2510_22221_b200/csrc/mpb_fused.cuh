// mpb_fused.cuh -- fused single-sweep variant (placeholder until written).
#pragma once
namespace {
int prepare_fused(mpb_handle*, const Geom&) {
    return fail_msg(MPB_EINVAL, "fused sweep not built in this version; use kernel_variant=1");
}
void destroy_fused(mpb_handle*) {}
int launch_fused(mpb_handle*, const Geom&, const Bufs&, cudaStream_t) { return MPB_EINVAL; }
int launch_deferred(mpb_handle*, const Geom&, const Bufs&, cudaStream_t) { return MPB_EINVAL; }
const char* fused_kernel_name() { return "none"; }
}  // namespace
