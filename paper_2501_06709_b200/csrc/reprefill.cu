// placeholder: tcgen05 re-prefill lands in the next milestone
#include "kvmig_common.cuh"
extern "C" int kvm_reprefill(const kvm_reprefill_args* args, void* stream) {
  (void)args; (void)stream;
  return kvm::fail(KVM_ERR_UNSUPPORTED, "kvm_reprefill not built yet");
}
