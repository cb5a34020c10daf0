// kvm_plan_hybrid — native restatement of the reference planner
// (/root/reference/pkg/src/kvpack/migration.py:128-170), SURVEY.md §8f row 4.
//
// Same decisions bit for bit: consensus order (-kv_bytes, item)
// (migration.py:128-134); per move, KV transfer if the link's comm budget
// still fits (:155-158), else re-prefill if the destination's compute budget
// fits (:159-163), else forced KV transfer after max_defer deferrals
// (:164-167), else deferred.  Ledgers are float64 and accumulate exactly as
// the reference's `used + int` (int converted to double, round-to-nearest),
// and are reported in first-use order (the reference's dict insertion order).

#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/kvmig.h"

namespace kvm {
int fail(int code, const std::string& msg);
}

namespace {

struct Ledger {
  std::vector<int64_t> keys;
  std::vector<double> used;
  int find(int64_t k) const {
    for (size_t i = 0; i < keys.size(); ++i)
      if (keys[i] == k) return (int)i;
    return -1;
  }
  double get(int64_t k) const {
    int i = find(k);
    return i < 0 ? 0.0 : used[i];
  }
  void set(int64_t k, double v) {
    int i = find(k);
    if (i < 0) {
      keys.push_back(k);
      used.push_back(v);
    } else {
      used[i] = v;
    }
  }
};

}  // namespace

extern "C" int kvm_plan_hybrid(const kvm_pending* moves, int n, const kvm_plan_params* pp, kvm_planned* out,
                               kvm_plan_ledgers* ledgers) {
  if (n < 0) return kvm::fail(KVM_ERR_INVALID, "n < 0");
  if (!pp || (n > 0 && (!moves || !out))) return kvm::fail(KVM_ERR_INVALID, "NULL argument");
  if (pp->gpus_per_machine < 1) return kvm::fail(KVM_ERR_CONFIG, "gpus_per_machine must be >= 1");
  if (!(pp->intra_bandwidth > 0) || !(pp->inter_bandwidth > 0) || !(pp->prefill_tokens_per_s > 0))
    return kvm::fail(KVM_ERR_CONFIG, "bandwidths and prefill rate must be > 0");
  if (pp->n_overrides < 0 || (pp->n_overrides > 0 && (!pp->override_link || !pp->override_budget)))
    return kvm::fail(KVM_ERR_INVALID, "bad comm-budget overrides");

  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    if (moves[a].kv_bytes != moves[b].kv_bytes) return moves[a].kv_bytes > moves[b].kv_bytes;
    return moves[a].item < moves[b].item;
  });

  // link key: machine id (>= 0) for ("intra", m), -1 for ("inter",)
  auto budget_of = [&](int64_t link) -> double {
    for (int i = 0; i < pp->n_overrides; ++i)
      if (pp->override_link[i] == link) return pp->override_budget[i];
    return link >= 0 ? pp->intra_comm_budget : pp->inter_comm_budget;
  };
  Ledger links, dests;
  for (int k = 0; k < n; ++k) {
    const int i = order[k];
    const kvm_pending& mv = moves[i];
    const int64_t ms = mv.src / pp->gpus_per_machine;
    const int64_t md = mv.dst / pp->gpus_per_machine;
    // Python floor division for negative ids (never produced by the reference) kept consistent:
    const int64_t fs = (mv.src < 0 && mv.src % pp->gpus_per_machine) ? ms - 1 : ms;
    const int64_t fd = (mv.dst < 0 && mv.dst % pp->gpus_per_machine) ? md - 1 : md;
    const int64_t link = (fs == fd) ? fs : -1;
    const double bw = link >= 0 ? pp->intra_bandwidth : pp->inter_bandwidth;
    const double used_link = links.get(link);
    const double used_dest = dests.get(mv.dst);
    kvm_planned& o = out[k];
    o.index = i;
    if (used_link + (double)mv.kv_bytes <= budget_of(link)) {
      links.set(link, used_link + (double)mv.kv_bytes);
      o.mode = KVM_MODE_KV_TRANSFER;
      o.latency_s = (double)mv.kv_bytes / bw;
    } else if (used_dest + (double)mv.tokens <= pp->comp_budget) {
      dests.set(mv.dst, used_dest + (double)mv.tokens);
      o.mode = KVM_MODE_TOKEN_TRANSFER;
      o.latency_s = (double)mv.tokens / pp->prefill_tokens_per_s;
    } else if (mv.defer_count >= pp->max_defer) {
      o.mode = KVM_MODE_FORCED_KV_TRANSFER;
      o.latency_s = (double)mv.kv_bytes / bw;
    } else {
      o.mode = KVM_MODE_DEFERRED;
      o.latency_s = 0.0;
    }
  }
  if (ledgers) {
    ledgers->n_links = (int32_t)links.keys.size();
    ledgers->n_dests = (int32_t)dests.keys.size();
    if (ledgers->capacity < (int32_t)std::max(links.keys.size(), dests.keys.size()))
      return kvm::fail(KVM_ERR_INVALID, "ledger capacity too small");
    for (size_t i = 0; i < links.keys.size(); ++i) {
      ledgers->link_key[i] = links.keys[i];
      ledgers->link_used[i] = links.used[i];
    }
    for (size_t i = 0; i < dests.keys.size(); ++i) {
      ledgers->dest_key[i] = dests.keys[i];
      ledgers->dest_used[i] = dests.used[i];
    }
  }
  return KVM_OK;
}
