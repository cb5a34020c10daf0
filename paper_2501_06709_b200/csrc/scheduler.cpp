// Native online scheduler: the reference's ClusterState (model.py:116-305) and
// MellScheduler (scheduler.py:217-1200) restated in C++ so the control plane
// that emits migration decisions runs at microseconds per slot instead of the
// reference's 1.6 ms, and so the GPU box can run the
// live loop without the reference installed.
//
// Decisions are meant to be identical to the reference's on every input: the
// same placement rules, the same tie-breaks ((priority, -gpu) maxima,
// (-size, id) item orders, lowest-free GPU id reuse, descending group ids),
// the same float64 priority arithmetic (free/capacity as a correctly rounded
// double division of exact integers, then w_free*frac - w_count*n; build with
// -ffp-contract=off so no FMA changes a rounding), and the same batched-epoch
// protocol (run sequential and batched on clones, adopt the batched outcome
// only if it needs no more migrations, scheduler.py:979-1007).  Parity is
// checked against the reference by tests/test_scheduler_native.py.
//
// Python-visible ordering: the reference's dicts iterate in insertion order;
// each entry here carries an insertion stamp so snapshots reproduce that order.

#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <array>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/kvmig.h"

namespace kvm {
int fail(int code, const std::string& msg);
}

namespace {

constexpr int64_t NONE = INT64_MIN;  // Python None for optional ids

enum Cls : int32_t { CL = KVM_CLASS_L, CM = KVM_CLASS_M, CS = KVM_CLASS_S, CT = KVM_CLASS_T, CTINY = KVM_CLASS_TINY };

struct Err {
  int code;
  std::string msg;
};
[[noreturn]] void raise(int code, const std::string& m) { throw Err{code, m}; }

// classify_request (model.py:72-86); 128-bit products so any int64 capacity works.
Cls classify(int64_t size, int64_t cap) {
  if (size <= 0) raise(KVM_ERR_INVALID, "size must be positive");
  if (size > cap)
    raise(KVM_ERR_TOO_LARGE, "size " + std::to_string(size) + " exceeds capacity " + std::to_string(cap));
  __int128 s = size, c = cap;
  if (2 * s > c) return CL;
  if (3 * s > c) return CM;
  if (4 * s > c) return CS;
  if (8 * s > c) return CT;
  return CTINY;
}

inline bool is_sm(Cls c) { return c == CM || c == CS; }
inline bool is_t(Cls c) { return c == CT || c == CTINY; }

// Per-GPU derived state, rebuilt lazily after any mutation that can change it
// (the reference keeps a similar family cache, model.py:138-139).
struct Summary {
  struct Entry {
    int64_t neg_size, id;
    int32_t cls;  // -1: size <= 0 (classifying it raises, as item_class does)
  };
  bool valid = false;
  int32_t fam = -2;  // -2: not computed yet
  int64_t used = 0, largest = 0, largest_id = INT64_MIN;
  std::vector<Entry> items;  // residents by (-size, id)
};

// Sorted small id set (GPU residents, group members): copies are one memcpy,
// which keeps the batched epoch's two cluster clones cheap (scheduler.py:993-994).
class IdSet {
 public:
  using const_iterator = std::vector<int64_t>::const_iterator;
  void insert(int64_t x) {
    auto it = std::lower_bound(v.begin(), v.end(), x);
    if (it == v.end() || *it != x) v.insert(it, x);
  }
  void erase(int64_t x) {
    auto it = std::lower_bound(v.begin(), v.end(), x);
    if (it != v.end() && *it == x) v.erase(it);
  }
  bool count(int64_t x) const { return std::binary_search(v.begin(), v.end(), x); }
  bool empty() const { return v.empty(); }
  size_t size() const { return v.size(); }
  const_iterator begin() const { return v.begin(); }
  const_iterator end() const { return v.end(); }

 private:
  std::vector<int64_t> v;
};

// Open-addressing int64 -> V map (linear probing, power-of-two table, load
// <= 1/2).  KVM_NONE and KVM_NONE + 1 are reserved as empty / tombstone keys.
template <class V>
class FlatMap {
 public:
  V* get(int64_t k) {
    if (keys.empty()) return nullptr;
    size_t m = keys.size() - 1;
    for (size_t i = hash(k) & m;; i = (i + 1) & m) {
      if (keys[i] == k) return &vals[i];
      if (keys[i] == EMPTY) return nullptr;
    }
  }
  const V* get(int64_t k) const { return const_cast<FlatMap*>(this)->get(k); }
  bool count(int64_t k) const { return get(k) != nullptr; }
  size_t size() const { return n; }
  // inserts a default value if missing; returns (value, inserted)
  std::pair<V*, bool> slot(int64_t k) {
    if (V* p = get(k)) return {p, false};
    if (2 * (n + dead + 1) > keys.size()) grow();
    size_t m = keys.size() - 1;
    for (size_t i = hash(k) & m;; i = (i + 1) & m) {
      if (keys[i] == EMPTY || keys[i] == DEAD) {
        if (keys[i] == DEAD) --dead;
        keys[i] = k;
        vals[i] = V();
        ++n;
        return {&vals[i], true};
      }
    }
  }
  V& operator[](int64_t k) { return *slot(k).first; }
  bool erase(int64_t k) {
    if (keys.empty()) return false;
    size_t m = keys.size() - 1;
    for (size_t i = hash(k) & m;; i = (i + 1) & m) {
      if (keys[i] == k) {
        keys[i] = DEAD;
        --n;
        ++dead;
        return true;
      }
      if (keys[i] == EMPTY) return false;
    }
  }
  template <class F>
  void each(F f) const {
    for (size_t i = 0; i < keys.size(); ++i)
      if (keys[i] != EMPTY && keys[i] != DEAD) f(keys[i], vals[i]);
  }

 private:
  static constexpr int64_t EMPTY = INT64_MIN, DEAD = INT64_MIN + 1;
  static size_t hash(int64_t k) { return (size_t)((uint64_t)k * 0x9E3779B97F4A7C15ull >> 17); }
  void grow() {
    std::vector<int64_t> ok = std::move(keys);
    std::vector<V> ov = std::move(vals);
    size_t cap = 16;
    while (cap < 4 * (n + 1)) cap <<= 1;
    keys.assign(cap, EMPTY);
    vals.assign(cap, V());
    n = dead = 0;
    for (size_t i = 0; i < ok.size(); ++i)
      if (ok[i] != EMPTY && ok[i] != DEAD) *slot(ok[i]).first = ov[i];
  }
  std::vector<int64_t> keys;
  std::vector<V> vals;
  size_t n = 0, dead = 0;
};

struct Gpu {
  int64_t machine = 0;
  int64_t seq = 0;
  uint64_t stamp = 0;
  IdSet residents;
  Summary sum;
};
struct Group {
  IdSet members;
  int64_t agg = 0;
  uint64_t stamp = 0;
};
struct Stamped {
  int64_t v = 0;
  uint64_t stamp = 0;
};

// Active GPUs by id.  Ids are dense (lowest-free reuse, model.py:191-197), so
// a vector indexed by id replaces the reference's dict; iteration is by id.
class GpuTable {
 public:
  struct Ref {
    int64_t first;
    Gpu& second;
  };
  struct It {
    GpuTable* t;
    int64_t i;
    void skip() {
      while (i < (int64_t)t->v.size() && !t->on[i]) ++i;
    }
    Ref operator*() const { return {i, t->v[i]}; }
    It& operator++() {
      ++i;
      skip();
      return *this;
    }
    bool operator!=(const It& o) const { return i != o.i; }
  };
  It begin() {
    It it{this, 0};
    it.skip();
    return it;
  }
  It end() { return It{this, (int64_t)v.size()}; }
  Gpu* find(int64_t g) { return (g >= 0 && g < (int64_t)v.size() && on[g]) ? &v[g] : nullptr; }
  const Gpu* find(int64_t g) const { return (g >= 0 && g < (int64_t)v.size() && on[g]) ? &v[g] : nullptr; }
  bool count(int64_t g) const { return find(g) != nullptr; }
  Gpu& insert(int64_t g, Gpu&& x) {
    if (g >= (int64_t)v.size()) {
      v.resize(g + 1);
      on.resize(g + 1, 0);
    }
    v[g] = std::move(x);
    on[g] = 1;
    return v[g];
  }
  void erase(int64_t g) {
    on[g] = 0;
    v[g] = Gpu();
  }

 private:
  std::vector<Gpu> v;
  std::vector<char> on;
};

// ---------------------------------------------------------------------------
// ClusterState (model.py:116-305)
// ---------------------------------------------------------------------------
struct Cluster {
  int64_t cap = 0;
  int64_t gpm = 4;
  GpuTable gpus;                                  // gpu id -> state
  FlatMap<Stamped> placement;                     // item -> gpu
  FlatMap<Stamped> sizes;                         // request -> bytes
  std::map<int64_t, Group> groups;                // gid (< 0) -> group
  FlatMap<Stamped> req_group;                     // request -> gid
  int64_t next_seq = 0;
  int64_t next_gid = -1;
  int64_t next_gpu = 0;
  std::set<int64_t> free_ids;  // the reference's min-heap of released ids
  uint64_t stamp = 0;
  uint64_t version = 0;
  // Family lists and latest-of-family per category, rebuilt when `dirt` moves
  // (any change to a GPU's residents, item sizes, activation or order).
  uint64_t dirt = 1;
  struct FamIndex {
    uint64_t at = 0;
    std::vector<int64_t> of[4];
    int64_t latest[4];
  } fidx;

  const Gpu& gpu(int64_t g) const {
    const Gpu* p = gpus.find(g);
    if (!p) raise(KVM_ERR_KEY, "GPU " + std::to_string(g) + " is not active");
    return *p;
  }
  Gpu& gpu(int64_t g) { return const_cast<Gpu&>(static_cast<const Cluster*>(this)->gpu(g)); }
  bool active(int64_t g) const { return g != NONE && gpus.count(g); }
  bool has_residents(int64_t g) const {
    const Gpu* p = gpus.find(g);
    return p && !p->residents.empty();
  }
  void touch(Gpu& g) {
    g.sum.valid = false;
    ++dirt;
  }

  // Invalidate the summary of the GPU hosting `item` (and of its group's host).
  void dirty_item(int64_t item) {
    if (const Stamped* h = placement.get(item)) {
      Gpu* p = gpus.find(h->v);
      if (p) touch(*p);
    }
    if (item >= 0) {
      if (const Stamped* rg = req_group.get(item)) dirty_item(rg->v);
    }
  }
  const Summary& summary(int64_t g) {
    Gpu& st = gpu(g);
    Summary& sm = st.sum;
    if (sm.valid) return sm;
    sm.items.clear();
    sm.used = 0;
    sm.largest = 0;
    sm.largest_id = INT64_MIN;
    sm.fam = -2;
    for (int64_t it : st.residents) {
      int64_t sz = item_size(it);
      sm.used += sz;
      if (sm.largest_id == INT64_MIN || sz > sm.largest || (sz == sm.largest && it > sm.largest_id))
        sm.largest = sz, sm.largest_id = it;
      int32_t k = -1;
      if (sz > 0) k = classify(std::min(sz, cap), cap);
      sm.items.push_back({-sz, it, k});
    }
    std::sort(sm.items.begin(), sm.items.end(),
              [](const Summary::Entry& a, const Summary::Entry& b) {
                return a.neg_size != b.neg_size ? a.neg_size < b.neg_size : a.id < b.id;
              });
    sm.valid = true;
    return sm;
  }

  int64_t size_of(int64_t r) const {
    const Stamped* p = sizes.get(r);
    if (!p) raise(KVM_ERR_KEY, "no size for request " + std::to_string(r));
    return p->v;
  }
  void put_size(int64_t r, int64_t v) {  // `sizes[r] = v` (keeps dict position)
    dirty_item(r);
    auto sl = sizes.slot(r);
    if (sl.second) sl.first->stamp = ++stamp;
    sl.first->v = v;
    ++version;
  }
  void del_size(int64_t r) {
    dirty_item(r);
    if (!sizes.erase(r)) raise(KVM_ERR_KEY, "no size for request " + std::to_string(r));
    ++version;
  }
  Group& group(int64_t gid) {
    auto it = groups.find(gid);
    if (it == groups.end()) raise(KVM_ERR_KEY, "no group " + std::to_string(gid));
    return it->second;
  }
  int64_t group_of(int64_t r) const {  // request_group.get(r) or NONE
    const Stamped* p = req_group.get(r);
    return p ? p->v : NONE;
  }

  // model.py:143-146
  int64_t item_size(int64_t item) {
    if (item < 0) return group(item).agg;
    return size_of(item);
  }
  // model.py:148-157
  void set_size(int64_t r, int64_t size) {
    dirty_item(r);
    int64_t old = size_of(r);
    put_size(r, size);
    int64_t gid = group_of(r);
    if (gid != NONE) group(gid).agg += size - old;
  }
  // model.py:159-175
  void group_add(int64_t gid, int64_t r) {
    dirty_item(gid);
    Group& g = group(gid);
    int64_t s = size_of(r);
    g.members.insert(r);
    g.agg += s;
    auto sl = req_group.slot(r);
    if (sl.second) sl.first->stamp = ++stamp;
    sl.first->v = gid;
    ++version;
  }
  void group_remove(int64_t gid, int64_t r) {
    dirty_item(gid);
    Group& g = group(gid);
    int64_t s = size_of(r);
    g.members.erase(r);
    g.agg -= s;
    req_group.erase(r);
    ++version;
  }
  void del_group(int64_t gid) {
    dirty_item(gid);
    if (!groups.erase(gid)) raise(KVM_ERR_KEY, "no group " + std::to_string(gid));
    ++version;
  }
  // model.py:177-181
  Cls item_class(int64_t item) { return classify(std::min(item_size(item), cap), cap); }
  int64_t used_bytes(int64_t g) { return summary(g).used; }
  int64_t free_bytes(int64_t g) { return cap - used_bytes(g); }
  bool conforms_threequarter(int64_t g) {  // scheduler.py:98-99
    return (__int128)4 * used_bytes(g) >= (__int128)3 * cap;
  }

  // model.py:191-219
  int64_t activate_gpu() {
    int64_t id;
    if (!free_ids.empty()) {
      id = *free_ids.begin();
      free_ids.erase(free_ids.begin());
    } else {
      id = next_gpu++;
    }
    Gpu g;
    g.machine = id / gpm;  // ids are non-negative
    g.seq = next_seq++;
    g.stamp = ++stamp;
    gpus.insert(id, std::move(g));
    ++version;
    ++dirt;
    return id;
  }
  void terminate_gpu(int64_t g) {
    Gpu* p = gpus.find(g);
    if (!p) raise(KVM_ERR_KEY, "GPU " + std::to_string(g) + " is not active");
    bool busy = !p->residents.empty();
    gpus.erase(g);  // the reference pops before it checks (model.py:210-212)
    ++version;
    ++dirt;
    if (busy) raise(KVM_ERR_INVALID, "GPU " + std::to_string(g) + " still has residents");
    free_ids.insert(g);
  }
  std::vector<int64_t> terminate_idle_gpus() {
    std::vector<int64_t> idle;
    for (auto kv : gpus)
      if (kv.second.residents.empty()) idle.push_back(kv.first);
    for (int64_t g : idle) terminate_gpu(g);
    return idle;
  }
  // model.py:223-239
  void place(int64_t item, int64_t g) {
    if (placement.count(item)) raise(KVM_ERR_INVALID, "item " + std::to_string(item) + " already placed");
    Gpu& st = gpu(g);
    st.residents.insert(item);
    touch(st);
    *placement.slot(item).first = Stamped{g, ++stamp};
    ++version;
  }
  int64_t unplace(int64_t item) {
    const Stamped* h = placement.get(item);
    if (!h) raise(KVM_ERR_NOT_FOUND, "item " + std::to_string(item) + " not placed");
    int64_t g = h->v;
    placement.erase(item);
    if (Gpu* p = gpus.find(g)) {
      p->residents.erase(item);
      touch(*p);
    }
    ++version;
    return g;
  }
  int64_t gpu_of(int64_t item) const {
    const Stamped* h = placement.get(item);
    return h ? h->v : NONE;
  }
  int64_t new_group() {
    int64_t gid = next_gid--;
    Group g;
    g.stamp = ++stamp;
    groups[gid] = std::move(g);
    ++version;
    return gid;
  }
  int64_t item_of_request(int64_t r) const {
    int64_t g = group_of(r);
    return g == NONE ? r : g;
  }
  // model.py:254-268: class of the largest resident (ties: larger id)
  Cls gpu_class(int64_t g) {
    if (gpu(g).residents.empty()) raise(KVM_ERR_NO_CATEGORY, "GPU " + std::to_string(g) + " is empty");
    const Summary& sm = summary(g);
    return classify(std::min(sm.largest, cap), cap);
  }
  Cls gpu_family(int64_t g) {
    Gpu& st = gpu(g);
    if (st.sum.valid && st.sum.fam >= 0) return (Cls)st.sum.fam;
    Cls c = gpu_class(g);
    c = c == CTINY ? CT : c;
    st.sum.fam = c;
    return c;
  }
  const FamIndex& fam_index() {
    if (fidx.at == dirt) return fidx;
    for (int f = 0; f < 4; ++f) fidx.of[f].clear(), fidx.latest[f] = NONE;
    int64_t seq[4] = {0, 0, 0, 0};
    for (auto kv : gpus) {
      if (kv.second.residents.empty()) continue;
      int f = gpu_family(kv.first);
      fidx.of[f].push_back(kv.first);
      if (fidx.latest[f] == NONE || kv.second.seq > seq[f]) fidx.latest[f] = kv.first, seq[f] = kv.second.seq;
    }
    fidx.at = dirt;
    return fidx;
  }
  std::vector<int64_t> gpus_of_family(Cls fam) { return fam_index().of[fam]; }  // ascending ids
  int64_t latest_of(const std::vector<int64_t>& cands) const {
    int64_t best = NONE, seq = 0;
    for (int64_t g : cands) {
      int64_t s = gpu(g).seq;
      if (best == NONE || s > seq) best = g, seq = s;
    }
    return best;
  }
  int64_t latest_gpu_of_family(Cls fam) { return fam_index().latest[fam]; }
  void check_capacity() {
    for (auto kv : gpus) {
      if (kv.second.residents.empty()) continue;
      int64_t u = used_bytes(kv.first);
      if (u > cap)
        raise(KVM_ERR_ASSERT, "GPU " + std::to_string(kv.first) + " over capacity: " + std::to_string(u) +
                                  " > " + std::to_string(cap));
    }
  }
};

// ---------------------------------------------------------------------------
// verify_properties (scheduler.py:102-191)
// ---------------------------------------------------------------------------
struct Violation {
  int64_t gpu;
  int32_t code;  // KVM_VIOLATION_*
};

std::vector<Violation> verify(Cluster& c, const std::set<int64_t>* exempt_in) {
  struct Info {
    int64_t g;
    Cls fam;
    int64_t used, largest, seq;
    int n[5];
  };
  std::vector<Info> info;  // non-empty GPUs, ascending id (the reference sorts, :159)
  const __int128 cap = c.cap;
  int64_t smallest_sm = INT64_MAX;  // smallest S/M item on an S/M-family GPU (:149-152)
  bool any_sm = false;
  for (auto kv : c.gpus) {
    if (kv.second.residents.empty()) continue;
    const Summary& sm = c.summary(kv.first);
    Info in{kv.first, CT, sm.used, 0, kv.second.seq, {0, 0, 0, 0, 0}};
    for (auto& e : sm.items) in.n[e.cls < 0 ? CTINY : e.cls]++;  // size <= 0 counts as Tiny (8*s <= C)
    in.largest = std::max<int64_t>(0, sm.largest);
    Cls fam = classify(std::min(in.largest, c.cap), c.cap);
    in.fam = fam == CTINY ? CT : fam;
    if (is_sm(in.fam))
      for (auto& e : sm.items)
        if (e.cls == CM || e.cls == CS) smallest_sm = std::min(smallest_sm, -e.neg_size), any_sm = true;
    info.push_back(in);
  }
  std::set<int64_t> exempt;
  if (exempt_in) {
    exempt = *exempt_in;
  } else {
    int64_t lg[4] = {NONE, NONE, NONE, NONE}, ls[4] = {0, 0, 0, 0};
    for (auto& in : info)
      if (lg[in.fam] == NONE || in.seq > ls[in.fam]) lg[in.fam] = in.g, ls[in.fam] = in.seq;
    for (int f = 0; f < 4; ++f)
      if (lg[f] != NONE) exempt.insert(lg[f]);
  }
  bool t_present = false;
  for (auto& in : info)
    if (in.fam == CT && !exempt.count(in.g)) t_present = true;
  std::vector<Violation> out;
  for (auto& in : info) {
    int64_t g = in.g;
    int total = in.n[0] + in.n[1] + in.n[2] + in.n[3] + in.n[4];
    if (in.used > c.cap) out.push_back({g, KVM_VIOLATION_CAPACITY});
    if (exempt.count(g)) continue;
    bool under = (__int128)4 * in.used < 3 * cap;
    if (in.fam == CM) {
      int nm = in.n[CM], nt = in.n[CT] + in.n[CTINY];
      if (nm != 2 || nt > 1 || nm + nt != total) out.push_back({g, KVM_VIOLATION_P1});
    } else if (in.fam == CS) {
      if (in.n[CS] != 3 || in.n[CS] != total) out.push_back({g, KVM_VIOLATION_P2});
    } else if (in.fam == CT) {
      if (under) out.push_back({g, KVM_VIOLATION_P3});
    } else if (in.fam == CL) {
      int nsm = in.n[CM] + in.n[CS];
      if (nsm == 0) {
        int64_t freeb = c.cap - in.used;
        int64_t limit = std::min(freeb, c.cap - in.largest - 1);
        if (any_sm && smallest_sm <= limit) out.push_back({g, KVM_VIOLATION_P4_MISSING});
      } else if (nsm > 1) {
        out.push_back({g, KVM_VIOLATION_P4_MULTIPLE});
      }
    }
    if (t_present && (in.fam == CL || in.fam == CM) && under) out.push_back({g, KVM_VIOLATION_P5});
  }
  return out;
}

// ---------------------------------------------------------------------------
// MellScheduler (scheduler.py:217-1200)
// ---------------------------------------------------------------------------
struct MoveRec {
  int64_t item, src, dst;
  int32_t reason;
};
struct Log {
  int32_t kind;
  int64_t request;
  std::vector<MoveRec> moves;
  std::vector<std::pair<int32_t, int64_t>> events;
  int64_t migrations() const {
    int64_t n = 0;
    for (auto& m : moves) n += m.src != NONE;
    return n;
  }
};
struct EpochOut {
  std::vector<Log> logs;
  std::vector<int64_t> terminated;
  bool batched = false;
  int64_t migrations() const {
    int64_t n = 0;
    for (auto& l : logs) n += l.migrations();
    return n;
  }
};

using Excl = std::vector<int64_t>;  // tiny exclude sets (0 or 1 ids)
inline bool in(const Excl& e, int64_t g) { return std::find(e.begin(), e.end(), g) != e.end(); }

struct Sched {
  Cluster* c;
  std::unique_ptr<Cluster> owned;  // clones own their cluster
  double w_free = 1.0, w_count = 0.25, w_same = 0.5;
  bool batching = false;
  FlatMap<int32_t> sched_class;  // item -> class at last decision
  std::vector<std::pair<int64_t, int64_t>> epoch_counts;

  int64_t cap() const { return c->cap; }

  // scheduler.py:68-84
  double alloc_prio(int64_t g) {
    volatile double frac = (double)c->free_bytes(g) / (double)c->cap;
    volatile double a = w_free * frac;
    volatile double b = w_count * (double)c->gpu(g).residents.size();
    return a - b;
  }
  double mig_prio(int64_t src, int64_t dst) {
    if (src == dst) raise(KVM_ERR_INVALID, "src and dst must differ");
    bool same = c->gpu(src).machine == c->gpu(dst).machine;
    volatile double p = alloc_prio(dst);
    volatile double add = w_same * (same ? 1.0 : 0.0);
    return p + add;
  }
  // max over (priority, -g): first strict improvement wins
  int64_t best_by_priority(const std::vector<int64_t>& ids) {
    int64_t best = NONE;
    double bp = 0;
    for (int64_t g : ids) {
      double p = alloc_prio(g);
      if (best == NONE || p > bp || (p == bp && -g > -best)) best = g, bp = p;
    }
    return best;
  }
  int64_t best_migration_peer(int64_t src, const std::vector<int64_t>& ids) {
    int64_t best = NONE;
    double bp = 0;
    for (int64_t g : ids) {
      double p = mig_prio(src, g);
      if (best == NONE || p > bp || (p == bp && -g > -best)) best = g, bp = p;
    }
    return best;
  }
  // scheduler.py:256-265
  int64_t fresh_gpu() {
    for (auto kv : c->gpus) {
      if (kv.second.residents.empty()) {
        kv.second.seq = c->next_seq++;
        ++c->version;
        ++c->dirt;
        return kv.first;
      }
    }
    return c->activate_gpu();
  }
  void record_place(int64_t item, int64_t g, Log& log, int32_t reason, int64_t src) {
    c->place(item, g);
    sched_class[item] = c->item_class(item);
    if (src != g) log.moves.push_back({item, src, g, reason});
  }
  void move(int64_t item, int64_t dst, Log& log, int32_t reason) {
    int64_t src = c->unplace(item);
    record_place(item, dst, log, reason, src);
  }
  // residents of the given classes, largest first, ties by id
  template <class Pred>
  std::vector<int64_t> items_where(int64_t g, Pred pred) {
    const Summary& sm = c->summary(g);
    std::vector<int64_t> out;
    for (auto& e : sm.items) {
      if (e.cls < 0) raise(KVM_ERR_INVALID, "size must be positive");
      if (pred((Cls)e.cls)) out.push_back(e.id);
    }
    return out;
  }
  template <class Pred>
  size_t count_where(int64_t g, Pred pred) {
    const Summary& sm = c->summary(g);
    size_t n = 0;
    for (auto& e : sm.items) {
      if (e.cls < 0) raise(KVM_ERR_INVALID, "size must be positive");
      n += pred((Cls)e.cls);
    }
    return n;
  }
  std::vector<int64_t> items_sm(int64_t g) { return items_where(g, is_sm); }
  size_t count_of(int64_t g, Cls k) {
    return count_where(g, [k](Cls x) { return x == k; });
  }
  std::vector<int64_t> items_t(int64_t g) { return items_where(g, is_t); }
  std::vector<int64_t> items_of(int64_t g, Cls k) {
    return items_where(g, [k](Cls x) { return x == k; });
  }
  int64_t latest_other(Cls fam, const Excl& ex) {
    std::vector<int64_t> cands;
    for (int64_t g : c->gpus_of_family(fam))
      if (!in(ex, g)) cands.push_back(g);
    return c->latest_of(cands);
  }
  std::array<int64_t, 4> latest_map() {
    return {c->latest_gpu_of_family(CL), c->latest_gpu_of_family(CM), c->latest_gpu_of_family(CS),
            c->latest_gpu_of_family(CT)};
  }

  // scheduler.py:297-318
  void repair_demoted(std::array<int64_t, 4> before, Log& log) {
    for (int round = 0; round < 3; ++round) {
      auto after = latest_map();
      std::set<int64_t> stale;
      for (int f = 0; f < 4; ++f) {
        int64_t old = before[f];
        if (old != NONE && after[f] != old && c->has_residents(old)) stale.insert(old);
      }
      if (stale.empty()) break;
      for (int64_t g : stale) repair_gpu(g, log);
      before = after;
    }
    ensure_l_coverage(log);
  }
  // scheduler.py:320-352
  void ensure_l_coverage(Log& log, int rounds = 3) {
    if (log.moves.size() < 2 && log.events.empty()) return;
    for (int r = 0; r < rounds; ++r) {
      int64_t smallest = NONE;
      for (Cls fam : {CM, CS})
        for (int64_t g : c->gpus_of_family(fam))
          for (int64_t it : items_sm(g)) {
            int64_t s = c->item_size(it);
            if (smallest == NONE || s < smallest) smallest = s;
          }
      if (smallest == NONE) return;
      int64_t exempt_l = c->latest_gpu_of_family(CL);
      bool pulled = false;
      for (int64_t g : c->gpus_of_family(CL)) {
        if (g == exempt_l || count_where(g, is_sm) != 0) continue;
        auto l_items = items_of(g, CL);
        if (l_items.empty()) raise(KVM_ERR_INVALID, "L-family GPU without an L item");
        int64_t limit = std::min(c->free_bytes(g), cap() - c->item_size(l_items[0]) - 1);
        if (smallest <= limit && pull_sm_to_l(g, log)) pulled = true;
      }
      if (!pulled) return;
    }
  }

  // scheduler.py:365-380
  void place_item(int64_t item, Log& log, int64_t src = NONE, const Excl& ex = {}, bool allow_evict = true,
                  bool prefer_holes = false, int32_t reason = KVM_REASON_ALLOCATE) {
    Cls cls = c->item_class(item);
    if (cls == CL)
      place_large(item, log, src, reason);
    else if (is_sm(cls))
      place_medium_small(item, cls, log, src, ex, allow_evict, prefer_holes, reason);
    else
      place_tiny_item(item, log, src, ex, prefer_holes, reason);
  }
  void place_large(int64_t item, Log& log, int64_t src, int32_t reason) {
    int64_t j = fresh_gpu();
    record_place(item, j, log, reason, src);
    if (!pull_sm_to_l(j, log)) fill_with_t(j, log);
  }
  // scheduler.py:390-425
  bool pull_sm_to_l(int64_t j, Log& log) {
    auto l_items = items_of(j, CL);
    if (l_items.empty()) return false;
    int64_t l_size = c->item_size(l_items[0]);
    int64_t freeb = c->free_bytes(j);
    auto fits = [&](int64_t it) {
      int64_t s = c->item_size(it);
      return l_size + s < cap() && s <= freeb;
    };
    std::vector<int64_t> donors;
    for (Cls fam : {CM, CS})
      for (int64_t d : c->gpus_of_family(fam)) {
        if (d == j) continue;
        for (int64_t it : items_sm(d))
          if (fits(it)) {
            donors.push_back(d);
            break;
          }
      }
    int64_t donor = best_migration_peer(j, donors);
    if (donor == NONE) return false;
    int64_t pick = NONE;
    for (int64_t it : items_sm(donor))
      if (fits(it)) {
        pick = it;
        break;
      }
    move(pick, j, log, KVM_REASON_L_FILL);
    if (c->has_residents(donor) && count_where(donor, is_sm) == 0) {
      for (int64_t t : items_t(donor)) {
        c->unplace(t);
        place_tiny_item(t, log, donor, {donor}, false, KVM_REASON_L_FILL);
      }
    } else {
      repair_gpu(donor, log);
    }
    return true;
  }
  // scheduler.py:427-446
  void fill_with_t(int64_t j, Log& log) {
    for (int i = 0; i < 8; ++i) {
      if (c->conforms_threequarter(j)) return;
      int64_t donor = c->latest_gpu_of_family(CT);
      if (donor == NONE || donor == j) return;
      int64_t freeb = c->free_bytes(j);
      int64_t pick = NONE;
      for (int64_t it : items_t(donor))
        if (c->item_size(it) <= freeb) {
          pick = it;
          break;
        }
      if (pick == NONE) return;
      move(pick, j, log, KVM_REASON_DEPART_REFILL);
    }
  }
  // scheduler.py:448-464
  void fill_m_with_t(int64_t j, Log& log) {
    if (!c->has_residents(j)) return;
    if (c->conforms_threequarter(j)) return;
    if (count_where(j, is_t) != 0) return;
    int64_t donor = latest_other(CT, {j});
    if (donor == NONE) return;
    int64_t freeb = c->free_bytes(j);
    for (int64_t it : items_t(donor))
      if (c->item_size(it) <= freeb) {
        move(it, j, log, KVM_REASON_DEPART_REFILL);
        return;
      }
  }
  // scheduler.py:466-524
  void place_medium_small(int64_t item, Cls cls, Log& log, int64_t src, const Excl& ex, bool allow_evict,
                          bool prefer_holes, int32_t reason) {
    int64_t size = c->item_size(item);
    auto l_candidates = [&](bool need_free) {
      std::vector<int64_t> out;
      for (int64_t g : c->gpus_of_family(CL)) {
        if (in(ex, g) || count_where(g, is_sm) != 0) continue;
        int64_t l_size = c->item_size(items_of(g, CL).at(0));
        if (l_size + size >= cap()) continue;
        if (need_free && c->free_bytes(g) < size) continue;
        out.push_back(g);
      }
      return out;
    };
    int64_t j = best_by_priority(l_candidates(true));
    if (j != NONE) {
      record_place(item, j, log, reason, src);
      return;
    }
    if (allow_evict) {
      j = best_by_priority(l_candidates(false));
      if (j != NONE) {
        place_with_t_eviction(item, j, log, src, reason);
        return;
      }
    }
    size_t slots = cls == CM ? 2 : 3;
    if (prefer_holes) {
      std::vector<int64_t> open;
      for (int64_t g : c->gpus_of_family(cls))
        if (!in(ex, g) && items_of(g, cls).size() < slots && c->free_bytes(g) >= size) open.push_back(g);
      j = best_by_priority(open);
      if (j != NONE) {
        record_place(item, j, log, reason, src);
        return;
      }
    }
    int64_t latest = latest_other(cls, ex);
    if (latest != NONE && items_of(latest, cls).size() < slots) {
      int64_t evictable = 0;
      for (int64_t t : items_t(latest)) evictable += c->item_size(t);
      if (c->free_bytes(latest) + evictable >= size) {
        place_with_t_eviction(item, latest, log, src, reason);
        if (cls == CM) fill_m_with_t(latest, log);
        return;
      }
    }
    int64_t was_latest = latest_other(cls, ex);
    j = fresh_gpu();
    record_place(item, j, log, reason, src);
    if (cls == CM && was_latest != NONE) fill_m_with_t(was_latest, log);
  }
  // scheduler.py:526-540
  void place_with_t_eviction(int64_t item, int64_t j, Log& log, int64_t src, int32_t reason) {
    int64_t size = c->item_size(item);
    std::vector<int64_t> evicted;
    for (int64_t t : items_t(j)) {
      if (c->free_bytes(j) >= size) break;
      c->unplace(t);
      evicted.push_back(t);
    }
    record_place(item, j, log, reason, src);
    for (int64_t t : evicted) place_tiny_item(t, log, j, {}, false, KVM_REASON_UPDATE);
  }
  // scheduler.py:542-567
  void place_tiny_item(int64_t item, Log& log, int64_t src, const Excl& ex, bool prefer_holes, int32_t reason) {
    int64_t size = c->item_size(item);
    std::vector<int64_t> cands;
    for (int64_t g : c->gpus_of_family(CL))
      if (!in(ex, g) && c->free_bytes(g) >= size) cands.push_back(g);
    int64_t j = best_by_priority(cands);
    if (j == NONE) {
      cands.clear();
      for (int64_t g : c->gpus_of_family(CM))
        if (!in(ex, g) && !c->conforms_threequarter(g) && count_where(g, is_t) == 0 && c->free_bytes(g) >= size)
          cands.push_back(g);
      j = best_by_priority(cands);
    }
    if (j == NONE && prefer_holes) {
      cands.clear();
      for (int64_t g : c->gpus_of_family(CT))
        if (!in(ex, g) && c->free_bytes(g) >= size) cands.push_back(g);
      j = best_by_priority(cands);
    }
    if (j == NONE) {
      int64_t latest = latest_other(CT, ex);
      if (latest != NONE && c->free_bytes(latest) >= size) j = latest;
    }
    if (j == NONE) j = fresh_gpu();
    record_place(item, j, log, reason, src);
  }
  void rehome_t_items(int64_t j, Log& log, int32_t reason, bool only_first) {
    for (int64_t t : items_t(j)) {
      c->unplace(t);
      place_tiny_item(t, log, j, {j}, false, reason);
      if (only_first) break;
    }
  }
  // scheduler.py:571-609
  void repair_gpu(int64_t j, Log& log) {
    if (!c->has_residents(j)) return;
    Cls fam = c->gpu_family(j);
    if (j == c->latest_gpu_of_family(fam)) return;
    if (fam == CL) {
      if (count_where(j, is_sm) == 0) pull_sm_to_l(j, log);
      if (!c->conforms_threequarter(j)) fill_with_t(j, log);
    } else if (fam == CM) {
      if (count_of(j, CM) < 2) refill_medium(j, log);
      fill_m_with_t(j, log);
    } else if (fam == CS) {
      rehome_t_items(j, log, KVM_REASON_DEPART_REFILL, false);
      while (count_of(j, CS) < 3) {
        int64_t donor = c->latest_gpu_of_family(CS);
        if (donor == NONE || donor == j) break;
        int64_t freeb = c->free_bytes(j);
        int64_t pick = NONE;
        for (int64_t it : items_of(donor, CS))
          if (c->item_size(it) <= freeb) {
            pick = it;
            break;
          }
        if (pick == NONE) break;
        move(pick, j, log, KVM_REASON_DEPART_REFILL);
      }
    } else {
      fill_with_t(j, log);
    }
  }
  // scheduler.py:611-637
  void refill_medium(int64_t j, Log& log) {
    int64_t donor = latest_other(CM, {j});
    if (donor == NONE) return;
    auto ms = items_of(donor, CM);
    auto first_fit = [&]() {
      int64_t freeb = c->free_bytes(j);
      for (int64_t it : ms)
        if (c->item_size(it) <= freeb) return it;
      return NONE;
    };
    int64_t pick = first_fit();
    if (pick == NONE) {
      rehome_t_items(j, log, KVM_REASON_DEPART_REFILL, true);
      pick = first_fit();
    }
    if (pick == NONE) return;
    move(pick, j, log, KVM_REASON_DEPART_REFILL);
    if (c->has_residents(donor) && count_of(donor, CM) == 0)
      rehome_t_items(donor, log, KVM_REASON_DEPART_REFILL, false);
  }

  // -- public operations (scheduler.py:641-876) ------------------------------
  Log allocate(int64_t r, int64_t size) {
    if (size > cap())
      raise(KVM_ERR_TOO_LARGE, "request " + std::to_string(r) + " needs " + std::to_string(size) + " > capacity " +
                                   std::to_string(cap()));
    if (size <= 0) raise(KVM_ERR_INVALID, "size must be positive");
    Log log{KVM_LOG_ALLOCATE, r, {}, {}};
    auto before = latest_map();
    c->put_size(r, size);
    if (classify(size, cap()) == CTINY)
      allocate_tiny(r, log);
    else
      place_item(r, log);
    repair_demoted(before, log);
    return log;
  }
  int64_t open_group(int64_t skip = NONE) {  // highest (least negative) open gid
    for (auto it = c->groups.rbegin(); it != c->groups.rend(); ++it)
      if (it->first != skip && (__int128)8 * it->second.agg <= cap()) return it->first;
    return NONE;
  }
  void allocate_tiny(int64_t r, Log& log) {
    int64_t gid = open_group();
    if (gid == NONE) {
      gid = c->new_group();
      c->group_add(gid, r);
      place_item(gid, log);
      return;
    }
    c->group_add(gid, r);
    int64_t j = c->gpu_of(gid);
    sched_class[gid] = c->item_class(gid);
    if (c->used_bytes(j) > cap()) {
      log.kind = KVM_LOG_UPDATE;
      c->unplace(gid);
      repair_gpu(j, log);
      place_item(gid, log, j, {j}, false, false, KVM_REASON_UPDATE);
    }
  }
  Log depart(int64_t r) {
    Log log{KVM_LOG_DEPART, r, {}, {}};
    auto before = latest_map();
    if (c->group_of(r) != NONE) {
      depart_group_member(r, log);
      repair_demoted(before, log);
      return log;
    }
    int64_t j = c->gpu_of(r);
    if (j == NONE) raise(KVM_ERR_NOT_FOUND, "request " + std::to_string(r) + " not placed");
    if (c->item_class(r) == CL) {
      depart_large(r, j, log);
    } else {
      c->unplace(r);
      sched_class.erase(r);
      c->del_size(r);
      repair_gpu(j, log);
    }
    repair_demoted(before, log);
    return log;
  }
  std::vector<int64_t> by_size_desc(const std::vector<int64_t>& items) {
    std::vector<std::pair<int64_t, int64_t>> v;
    for (int64_t it : items) v.push_back({-c->item_size(it), it});
    std::sort(v.begin(), v.end());
    std::vector<int64_t> out;
    for (auto& p : v) out.push_back(p.second);
    return out;
  }
  void depart_large(int64_t item, int64_t j, Log& log) {
    c->unplace(item);
    sched_class.erase(item);
    c->del_size(item);
    const auto& res = c->gpu(j).residents;
    auto others = by_size_desc(std::vector<int64_t>(res.begin(), res.end()));
    for (int64_t o : others) c->unplace(o);
    for (int64_t o : others) place_item(o, log, j, {}, false, false, KVM_REASON_DEPART_REFILL);
  }
  void drop_group(int64_t gid) {
    c->unplace(gid);
    sched_class.erase(gid);
    c->del_group(gid);
  }
  void depart_group_member(int64_t r, Log& log) {
    int64_t gid = c->group_of(r);
    c->group_remove(gid, r);
    c->del_size(r);
    int64_t j = c->gpu_of(gid);
    if (c->group(gid).members.empty()) {
      drop_group(gid);
      repair_gpu(j, log);
      return;
    }
    if ((__int128)8 * c->item_size(gid) <= cap()) {
      log.kind = KVM_LOG_UPDATE;
      reopen_group(gid, j, log);
    } else {
      sched_class[gid] = c->item_class(gid);
      repair_gpu(j, log);
    }
  }
  // scheduler.py:740-772
  void reopen_group(int64_t gid, int64_t j, Log& log) {
    int64_t other = open_group(gid);
    if (other != NONE) {
      int64_t dst_gpu = c->gpu_of(other);
      std::vector<int64_t> members(c->group(gid).members.begin(), c->group(gid).members.end());
      for (int64_t r : members) {
        c->group_remove(gid, r);
        c->group_add(other, r);
      }
      drop_group(gid);
      if (j != dst_gpu) log.moves.push_back({gid, j, dst_gpu, KVM_REASON_UPDATE});
      sched_class[other] = c->item_class(other);
      if (c->used_bytes(dst_gpu) > cap()) {
        int64_t src2 = c->unplace(other);
        repair_gpu(src2, log);
        place_item(other, log, src2, {src2}, false, false, KVM_REASON_UPDATE);
      }
      repair_gpu(j, log);
    } else {
      c->unplace(gid);
      repair_gpu(j, log);
      place_item(gid, log, j, {}, false, false, KVM_REASON_UPDATE);
    }
  }
  // scheduler.py:774-814
  Log update(int64_t r) {
    Log log{KVM_LOG_UPDATE, r, {}, {}};
    int64_t item = c->item_of_request(r);
    int64_t j = c->gpu_of(item);
    if (j == NONE) raise(KVM_ERR_NOT_FOUND, "request " + std::to_string(r) + " not placed");
    auto before = latest_map();
    const int32_t* oc = sched_class.get(item);
    int32_t old_cls = oc ? *oc : -1;
    Cls new_cls = c->item_class(item);
    if (new_cls == old_cls) {
      if (c->used_bytes(j) > cap()) resolve_overload(j, item, log);
      repair_demoted(before, log);
      return log;
    }
    if (new_cls == CL) {
      bool other_l = false;
      for (int64_t it : items_of(j, CL)) other_l |= it != item;
      if (other_l) {
        c->unplace(item);
        repair_gpu(j, log);
        place_item(item, log, j, {}, false, false, KVM_REASON_UPDATE);
      } else {
        sched_class[item] = new_cls;
        if (c->used_bytes(j) > cap()) resolve_overload(j, item, log);
        repair_gpu(j, log);
        int64_t demoted = latest_other(CL, {j});
        if (demoted != NONE) repair_gpu(demoted, log);
      }
    } else {
      c->unplace(item);
      repair_gpu(j, log);
      place_item(item, log, j, {}, false, false, KVM_REASON_UPDATE);
    }
    repair_demoted(before, log);
    return log;
  }
  // scheduler.py:816-848
  void resolve_overload(int64_t j, int64_t keep, Log& log) {
    std::vector<int64_t> rest;
    for (int64_t it : c->gpu(j).residents)
      if (it != keep) rest.push_back(it);
    auto others = by_size_desc(rest);
    for (int64_t o : others) c->unplace(o);
    for (int64_t o : others) place_item(o, log, j, {j}, false, false, KVM_REASON_UPDATE);
    if (c->gpu_of(keep) == j && is_sm(c->item_class(keep))) {
      int64_t dst = free_l_gpu_for(keep, {j});
      if (dst != NONE) move(keep, dst, log, KVM_REASON_UPDATE);
    }
    repair_gpu(j, log);
  }
  int64_t free_l_gpu_for(int64_t item, const Excl& ex) {
    int64_t size = c->item_size(item);
    std::vector<int64_t> cands;
    for (int64_t g : c->gpus_of_family(CL)) {
      if (in(ex, g) || count_where(g, is_sm) != 0) continue;
      int64_t l_size = c->item_size(items_of(g, CL).at(0));
      if (l_size + size < cap() && c->free_bytes(g) >= size) cands.push_back(g);
    }
    return best_by_priority(cands);
  }
  // scheduler.py:852-876
  void handle_growth(std::vector<int64_t> grown, std::vector<Log>& logs) {
    std::sort(grown.begin(), grown.end());
    for (int64_t r : grown) {
      if (c->group_of(r) != NONE) {
        Log log{KVM_LOG_UPDATE, r, {}, {}};
        if (group_member_growth(r, log)) logs.push_back(std::move(log));
        continue;
      }
      int64_t j = c->gpu_of(r);
      if (j == NONE) continue;
      if (c->size_of(r) > cap()) {
        logs.push_back(abort_request(r));
        continue;
      }
      const int32_t* oc = sched_class.get(r);
      int32_t old_cls = oc ? *oc : -1;
      if (old_cls != c->item_class(r) || c->used_bytes(j) > cap()) logs.push_back(update(r));
    }
  }
  Log abort_request(int64_t r) {
    Log log{KVM_LOG_UPDATE, r, {}, {}};
    auto before = latest_map();
    int64_t j = c->unplace(r);
    sched_class.erase(r);
    c->del_size(r);
    log.events.push_back({KVM_EVENT_ABORTED, r});
    repair_gpu(j, log);
    repair_demoted(before, log);
    return log;
  }
  // scheduler.py:890-942; returns whether a log was produced
  bool group_member_growth(int64_t r, Log& log) {
    int64_t gid = c->group_of(r);
    int64_t j = c->gpu_of(gid);
    auto before = latest_map();
    __int128 sr = c->size_of(r);
    if (sr > cap()) {
      c->group_remove(gid, r);
      c->del_size(r);
      log.events.push_back({KVM_EVENT_ABORTED, r});
      if (c->group(gid).members.empty()) drop_group(gid);
      if (c->has_residents(j)) repair_gpu(j, log);
      repair_demoted(before, log);
      return true;
    }
    if (8 * sr > cap()) {
      c->group_remove(gid, r);
      if (c->group(gid).members.empty())
        drop_group(gid);
      else if ((__int128)8 * c->item_size(gid) <= cap())
        reopen_group(gid, j, log);
      else
        sched_class[gid] = c->item_class(gid);
      Excl ex;
      if (c->active(j) && c->used_bytes(j) > cap()) ex.push_back(j);
      place_item(r, log, j, ex, false, false, KVM_REASON_UPDATE);
      if (c->has_residents(j)) repair_gpu(j, log);
      repair_demoted(before, log);
      return true;
    }
    if ((__int128)4 * c->item_size(gid) > cap()) {
      shed_group_members(gid, j, log);
      repair_demoted(before, log);
      return true;
    }
    if (c->used_bytes(j) > cap()) {
      resolve_overload(j, gid, log);
      repair_demoted(before, log);
      return true;
    }
    sched_class[gid] = c->item_class(gid);
    return false;
  }
  // scheduler.py:944-975
  void shed_group_members(int64_t gid, int64_t j, Log& log) {
    std::vector<std::pair<int64_t, int64_t>> order;  // (size, id) ascending
    for (int64_t r : c->group(gid).members) order.push_back({c->size_of(r), r});
    std::sort(order.begin(), order.end());
    std::vector<int64_t> shed;
    for (auto& p : order) {
      if ((__int128)4 * c->item_size(gid) <= cap()) break;
      c->group_remove(gid, p.second);
      shed.push_back(p.second);
    }
    sched_class[gid] = c->item_class(gid);
    int64_t open = open_group();
    if (open != NONE && open != gid) {
      int64_t dst = c->gpu_of(open);
      for (int64_t r : shed) {
        c->group_add(open, r);
        if (dst != j) log.moves.push_back({r, j, dst, KVM_REASON_UPDATE});
      }
      sched_class[open] = c->item_class(open);
      if (c->used_bytes(dst) > cap()) resolve_overload(dst, open, log);
    } else {
      int64_t ng = c->new_group();
      for (int64_t r : shed) c->group_add(ng, r);
      place_item(ng, log, j, {}, false, false, KVM_REASON_UPDATE);
    }
    if (c->active(j) && c->used_bytes(j) > cap())
      resolve_overload(j, gid, log);
    else if (c->has_residents(j))
      repair_gpu(j, log);
  }

  // -- epochs (scheduler.py:979-1176) -----------------------------------------
  struct Inputs {
    std::vector<std::pair<int64_t, int64_t>> arrivals;  // sorted
    std::vector<int64_t> completions;                   // sorted
    std::vector<std::pair<int64_t, int64_t>> growths;   // sorted by id, unique ids
  };
  EpochOut step_sequential(const Inputs& in) {
    EpochOut out;
    for (auto& g : in.growths)
      if (c->sizes.count(g.first)) c->set_size(g.first, std::max(c->size_of(g.first), g.second));
    for (int64_t r : in.completions) out.logs.push_back(depart(r));
    std::vector<int64_t> grown;
    for (auto& g : in.growths) grown.push_back(g.first);
    handle_growth(grown, out.logs);
    for (auto& a : in.arrivals) {
      try {
        out.logs.push_back(allocate(a.first, a.second));
      } catch (const Err& e) {
        if (e.code != KVM_ERR_TOO_LARGE) throw;
        Log log{KVM_LOG_ALLOCATE, a.first, {}, {}};
        log.events.push_back({KVM_EVENT_REJECTED, a.first});
        out.logs.push_back(std::move(log));
      }
    }
    out.terminated = c->terminate_idle_gpus();
    return out;
  }
  bool step_batched(const Inputs& in, EpochOut& out) {
    Log log{KVM_LOG_EPOCH, NONE, {}, {}};
    // phase 1: departs without refills
    for (int64_t r : in.completions) {
      int64_t gid = c->group_of(r);
      if (gid != NONE) {
        c->group_remove(gid, r);
        c->del_size(r);
        if (c->group(gid).members.empty()) drop_group(gid);
        continue;
      }
      if (c->gpu_of(r) == NONE) continue;
      c->unplace(r);
      sched_class.erase(r);
      c->del_size(r);
    }
    // phase 2: growth, aborts, members leaving groups
    for (auto& g : in.growths)
      if (c->sizes.count(g.first)) c->set_size(g.first, std::max(c->size_of(g.first), g.second));
    for (auto& g : in.growths) {
      int64_t r = g.first;
      int64_t gid = c->group_of(r);
      if (gid != NONE) {
        __int128 sr = c->size_of(r);
        if (sr > cap()) {
          c->group_remove(gid, r);
          c->del_size(r);
          log.events.push_back({KVM_EVENT_ABORTED, r});
          if (c->group(gid).members.empty()) drop_group(gid);
          continue;
        }
        if (8 * sr > cap()) {
          int64_t j = c->gpu_of(gid);
          c->group_remove(gid, r);
          if (c->group(gid).members.empty()) drop_group(gid);
          place_item(r, log, j, {}, false, true, KVM_REASON_UPDATE);
        }
      } else if (c->sizes.count(r) && c->gpu_of(r) != NONE) {
        if (c->size_of(r) > cap()) {
          c->unplace(r);
          sched_class.erase(r);
          c->del_size(r);
          log.events.push_back({KVM_EVENT_ABORTED, r});
        }
      }
    }
    // phase 3: allocates may consume the holes
    for (auto& a : in.arrivals) {
      if (a.second > cap()) {
        log.events.push_back({KVM_EVENT_REJECTED, a.first});
        continue;
      }
      c->put_size(a.first, a.second);
      if (classify(a.second, cap()) == CTINY)
        allocate_tiny(a.first, log);
      else
        place_item(a.first, log, NONE, {}, true, true, KVM_REASON_ALLOCATE);
    }
    // phase 4: global repair
    if (!repair_all(log)) return false;
    out.terminated = c->terminate_idle_gpus();
    if (!verify(*c, nullptr).empty()) return false;
    out.logs.push_back(std::move(log));
    out.batched = true;
    return true;
  }
  bool repair_all(Log& log) {
    for (int it = 0; it < 6; ++it) {
      bool changed = false;
      size_t before = log.moves.size();
      std::vector<int64_t> gids;
      for (auto g = c->groups.rbegin(); g != c->groups.rend(); ++g) gids.push_back(g->first);
      for (int64_t gid : gids)
        if ((__int128)4 * c->item_size(gid) > cap()) shed_group_members(gid, c->gpu_of(gid), log);
      std::vector<std::pair<int64_t, int64_t>> ord;
      for (auto kv : c->gpus)
        if (!kv.second.residents.empty()) ord.push_back({kv.second.seq, kv.first});
      std::sort(ord.begin(), ord.end());
      for (auto& p : ord) {
        int64_t j = p.second;
        if (!c->has_residents(j)) continue;
        if (c->used_bytes(j) > cap()) {
          int64_t keep = NONE, ks = 0;
          for (int64_t x : c->gpu(j).residents) {
            int64_t s = c->item_size(x);
            if (keep == NONE || s > ks || (s == ks && x > keep)) keep = x, ks = s;
          }
          resolve_overload(j, keep, log);
          changed = true;
        }
      }
      for (auto& p : ord) {
        int64_t j = p.second;
        if (!c->has_residents(j)) continue;
        if (repair_shape(j, log)) changed = true;
      }
      changed = changed || log.moves.size() > before;
      if (!changed && verify(*c, nullptr).empty()) return true;
    }
    return verify(*c, nullptr).empty();
  }
  void rehome_all(const std::vector<int64_t>& items, int64_t j, Log& log) {
    for (int64_t it : items) {
      c->unplace(it);
      place_item(it, log, j, {j}, false, true, KVM_REASON_BATCH);
    }
  }
  static std::vector<int64_t> tail(std::vector<int64_t> v, size_t from) {
    if (v.size() <= from) return {};
    return std::vector<int64_t>(v.begin() + from, v.end());
  }
  bool repair_shape(int64_t j, Log& log) {
    if (!c->has_residents(j)) return false;
    size_t before = log.moves.size();
    Cls fam = c->gpu_family(j);
    if (j == c->latest_gpu_of_family(fam)) return false;
    if (fam == CL) {
      rehome_all(tail(items_sm(j), 1), j, log);
    } else if (fam == CM) {
      rehome_all(items_of(j, CS), j, log);
      rehome_all(tail(items_of(j, CM), 2), j, log);
      rehome_all(tail(items_t(j), 1), j, log);
    } else if (fam == CS) {
      rehome_all(items_t(j), j, log);
      rehome_all(tail(items_of(j, CS), 3), j, log);
    }
    repair_gpu(j, log);
    return log.moves.size() > before;
  }

  void adopt(Sched& w) {
    // the reference swaps the winner's containers into self.cluster (:1187-1200)
    Cluster& d = *c;
    Cluster& s = *w.c;
    d.gpus = std::move(s.gpus);
    d.placement = std::move(s.placement);
    d.sizes = std::move(s.sizes);
    d.groups = std::move(s.groups);
    d.req_group = std::move(s.req_group);
    d.next_seq = s.next_seq;
    d.next_gid = s.next_gid;
    d.free_ids = std::move(s.free_ids);
    d.next_gpu = s.next_gpu;
    d.stamp = std::max(d.stamp, s.stamp);
    d.dirt = std::max(d.dirt, s.dirt) + 1;
    ++d.version;
    sched_class = std::move(w.sched_class);
  }
  std::unique_ptr<Sched> clone() const {
    auto o = std::make_unique<Sched>();
    o->owned = std::make_unique<Cluster>(*c);
    o->c = o->owned.get();
    o->w_free = w_free, o->w_count = w_count, o->w_same = w_same;
    o->batching = false;
    o->sched_class = sched_class;
    return o;
  }
  EpochOut step_epoch(const Inputs& in) {
    if (!batching) {
      EpochOut r = step_sequential(in);
      c->check_capacity();
      return r;
    }
    auto seq = clone();
    auto bat = clone();
    EpochOut sr = seq->step_sequential(in);
    EpochOut br;
    bool ok = bat->step_batched(in, br) && br.migrations() <= sr.migrations();
    EpochOut& res = ok ? br : sr;
    epoch_counts.push_back({sr.migrations(), res.migrations()});
    adopt(ok ? *bat : *seq);
    c->check_capacity();
    return std::move(res);
  }
};

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
struct kvm_cluster {
  Cluster c;
  std::vector<int64_t> buf;  // last snapshot / list result
};
struct kvm_sched {
  Sched s;
  std::vector<int64_t> buf;  // last result records
};

namespace {
template <class F>
int guard(F&& f) {
  try {
    return f();
  } catch (const Err& e) {
    return kvm::fail(e.code, e.msg);
  } catch (const std::exception& e) {
    return kvm::fail(KVM_ERR_INVALID, e.what());
  }
}
void emit(std::vector<int64_t>& b, int64_t tag, int64_t a, int64_t x = 0, int64_t y = 0, int64_t z = 0) {
  b.insert(b.end(), {tag, a, x, y, z});
}
void emit_logs(std::vector<int64_t>& b, const std::vector<Log>& logs) {
  for (auto& l : logs) {
    emit(b, KVM_REC_LOG, l.kind, l.request);
    for (auto& m : l.moves) emit(b, KVM_REC_MOVE, m.item, m.src, m.dst, m.reason);
    for (auto& e : l.events) emit(b, KVM_REC_EVENT, e.first, e.second);
  }
}
}  // namespace

extern "C" {

int kvm_cluster_create(int64_t capacity_bytes, int64_t gpus_per_machine, kvm_cluster** out) {
  return guard([&] {
    if (!out) raise(KVM_ERR_INVALID, "out is NULL");
    if (capacity_bytes <= 0) raise(KVM_ERR_INVALID, "capacity_bytes must be > 0");
    if (gpus_per_machine < 1) raise(KVM_ERR_INVALID, "gpus_per_machine must be >= 1");
    auto* h = new kvm_cluster();
    h->c.cap = capacity_bytes;
    h->c.gpm = gpus_per_machine;
    *out = h;
    return KVM_OK;
  });
}

void kvm_cluster_destroy(kvm_cluster* h) { delete h; }

int kvm_cluster_op(kvm_cluster* h, int op, int64_t a, int64_t b, int64_t* ret) {
  return guard([&] {
    if (!h) raise(KVM_ERR_INVALID, "cluster handle is NULL");
    Cluster& c = h->c;
    int64_t r = 0;
    switch (op) {
      case KVM_CL_ACTIVATE_GPU: r = c.activate_gpu(); break;
      case KVM_CL_TERMINATE_GPU: c.terminate_gpu(a); break;
      case KVM_CL_PLACE: c.place(a, b); break;
      case KVM_CL_UNPLACE: r = c.unplace(a); break;
      case KVM_CL_GPU_OF: r = c.gpu_of(a); break;
      case KVM_CL_SET_SIZE: c.set_size(a, b); break;
      case KVM_CL_PUT_SIZE: c.put_size(a, b); break;
      case KVM_CL_DEL_SIZE: c.del_size(a); break;
      case KVM_CL_NEW_GROUP: r = c.new_group(); break;
      case KVM_CL_GROUP_ADD: c.group_add(a, b); break;
      case KVM_CL_GROUP_REMOVE: c.group_remove(a, b); break;
      case KVM_CL_DEL_GROUP: c.del_group(a); break;
      case KVM_CL_ITEM_SIZE: r = c.item_size(a); break;
      case KVM_CL_ITEM_CLASS: r = c.item_class(a); break;
      case KVM_CL_USED_BYTES: r = c.used_bytes(a); break;
      case KVM_CL_GPU_CLASS: r = c.gpu_class(a); break;
      case KVM_CL_GPU_FAMILY: r = c.gpu_family(a); break;
      case KVM_CL_LATEST_OF_FAMILY: r = c.latest_gpu_of_family((Cls)a); break;
      case KVM_CL_CHECK_CAPACITY: c.check_capacity(); break;
      case KVM_CL_ITEM_OF_REQUEST: r = c.item_of_request(a); break;
      case KVM_CL_SET_ACTIVATION_SEQ: c.gpu(a).seq = b; ++c.version; ++c.dirt; break;
      case KVM_CL_SET_NEXT_ACTIVATION_SEQ: c.next_seq = a; ++c.version; break;
      case KVM_CL_VERSION: r = (int64_t)c.version; break;
      case KVM_CL_CLASSIFY: r = classify(a, b); break;
      case KVM_CL_VERSION_ADDR: r = (int64_t)(uintptr_t)&c.version; break;
      default: raise(KVM_ERR_INVALID, "unknown cluster op " + std::to_string(op));
    }
    if (ret) *ret = r;
    return KVM_OK;
  });
}

int kvm_cluster_terminate_idle(kvm_cluster* h, const int64_t** ids, int64_t* n) {
  return guard([&] {
    if (!h || !ids || !n) raise(KVM_ERR_INVALID, "NULL argument");
    auto idle = h->c.terminate_idle_gpus();
    h->buf.assign(idle.begin(), idle.end());
    *ids = h->buf.data();
    *n = (int64_t)h->buf.size();
    return KVM_OK;
  });
}

int kvm_cluster_snapshot(kvm_cluster* h, const int64_t** recs, int64_t* n) {
  return guard([&] {
    if (!h || !recs || !n) raise(KVM_ERR_INVALID, "NULL argument");
    Cluster& c = h->c;
    auto& b = h->buf;
    b.clear();
    emit(b, KVM_SNAP_COUNTERS, c.next_seq, c.next_gid, c.next_gpu, (int64_t)c.version);
    // dict contents in insertion order (stamps)
    std::vector<std::pair<uint64_t, int64_t>> ord;
    for (auto kv : c.gpus) ord.push_back({kv.second.stamp, kv.first});
    std::sort(ord.begin(), ord.end());
    for (auto& p : ord) {
      const Gpu& g = c.gpu(p.second);
      emit(b, KVM_SNAP_GPU, p.second, g.machine, g.seq, (int64_t)g.residents.size());
      for (int64_t it : g.residents) emit(b, KVM_SNAP_RESIDENT, it);
    }
    ord.clear();
    std::vector<std::tuple<uint64_t, int64_t, int64_t>> kv3;  // (stamp, key, value)
    auto dump = [&](const FlatMap<Stamped>& m, int64_t tag) {
      kv3.clear();
      m.each([&](int64_t k, const Stamped& x) { kv3.emplace_back(x.stamp, k, x.v); });
      std::sort(kv3.begin(), kv3.end());
      for (auto& t : kv3) emit(b, tag, std::get<1>(t), std::get<2>(t));
    };
    dump(c.placement, KVM_SNAP_PLACEMENT);
    dump(c.sizes, KVM_SNAP_SIZE);
    ord.clear();
    for (auto& kv : c.groups) ord.push_back({kv.second.stamp, kv.first});
    std::sort(ord.begin(), ord.end());
    for (auto& p : ord) {
      const Group& g = c.groups[p.second];
      emit(b, KVM_SNAP_GROUP, p.second, g.agg, (int64_t)g.members.size());
      for (int64_t m : g.members) emit(b, KVM_SNAP_MEMBER, m);
    }
    dump(c.req_group, KVM_SNAP_REQUEST_GROUP);
    for (int64_t g : c.free_ids) emit(b, KVM_SNAP_FREE_ID, g);
    *recs = b.data();
    *n = (int64_t)b.size() / 5;
    return KVM_OK;
  });
}

int kvm_cluster_verify(kvm_cluster* h, const int64_t* exempt, int64_t n_exempt, const int64_t** recs, int64_t* n) {
  return guard([&] {
    if (!h || !recs || !n) raise(KVM_ERR_INVALID, "NULL argument");
    std::set<int64_t> ex;
    if (n_exempt >= 0)
      for (int64_t i = 0; i < n_exempt; ++i) ex.insert(exempt[i]);
    auto v = verify(h->c, n_exempt >= 0 ? &ex : nullptr);
    h->buf.clear();
    for (auto& x : v) h->buf.insert(h->buf.end(), {x.gpu, (int64_t)x.code});
    *recs = h->buf.data();
    *n = (int64_t)v.size();
    return KVM_OK;
  });
}

int kvm_sched_create(kvm_cluster* cluster, const kvm_sched_params* p, kvm_sched** out) {
  return guard([&] {
    if (!cluster || !p || !out) raise(KVM_ERR_INVALID, "NULL argument");
    if (p->weight_free_mem < 0 || p->weight_request_count < 0 || p->weight_same_machine < 0)
      raise(KVM_ERR_INVALID, "priority weights must be non-negative");
    if (!(p->weight_free_mem != 0 || p->weight_request_count != 0 || p->weight_same_machine != 0))
      raise(KVM_ERR_INVALID, "at least one priority weight must be > 0");
    auto* h = new kvm_sched();
    h->s.c = &cluster->c;
    h->s.w_free = p->weight_free_mem;
    h->s.w_count = p->weight_request_count;
    h->s.w_same = p->weight_same_machine;
    h->s.batching = p->batching != 0;
    *out = h;
    return KVM_OK;
  });
}

void kvm_sched_destroy(kvm_sched* h) { delete h; }

int kvm_sched_set_batching(kvm_sched* h, int batching) {
  return guard([&] {
    if (!h) raise(KVM_ERR_INVALID, "NULL argument");
    h->s.batching = batching != 0;
    return KVM_OK;
  });
}

int kvm_sched_step_epoch(kvm_sched* h, const int64_t* arrivals, int64_t n_arr, const int64_t* completions,
                         int64_t n_comp, const int64_t* growths, int64_t n_grow, const int64_t** recs, int64_t* n) {
  return guard([&] {
    if (!h || !recs || !n) raise(KVM_ERR_INVALID, "NULL argument");
    Sched::Inputs in;
    for (int64_t i = 0; i < n_arr; ++i) in.arrivals.push_back({arrivals[2 * i], arrivals[2 * i + 1]});
    for (int64_t i = 0; i < n_comp; ++i) in.completions.push_back(completions[i]);
    for (int64_t i = 0; i < n_grow; ++i) in.growths.push_back({growths[2 * i], growths[2 * i + 1]});
    std::sort(in.arrivals.begin(), in.arrivals.end());
    std::sort(in.completions.begin(), in.completions.end());
    std::sort(in.growths.begin(), in.growths.end());
    for (size_t i = 1; i < in.growths.size(); ++i)
      if (in.growths[i].first == in.growths[i - 1].first) raise(KVM_ERR_INVALID, "duplicate growth id");
    size_t before = h->s.epoch_counts.size();
    EpochOut r = h->s.step_epoch(in);
    auto& b = h->buf;
    b.clear();
    emit_logs(b, r.logs);
    for (int64_t g : r.terminated) emit(b, KVM_REC_TERMINATED, g);
    emit(b, KVM_REC_BATCHED, r.batched ? 1 : 0);
    if (h->s.epoch_counts.size() > before)
      emit(b, KVM_REC_EPOCH_COUNTS, h->s.epoch_counts.back().first, h->s.epoch_counts.back().second);
    *recs = b.data();
    *n = (int64_t)b.size() / 5;
    return KVM_OK;
  });
}

int kvm_sched_op(kvm_sched* h, int op, const int64_t* ids, int64_t n_ids, int64_t size, const int64_t** recs,
                 int64_t* n) {
  return guard([&] {
    if (!h || !recs || !n) raise(KVM_ERR_INVALID, "NULL argument");
    std::vector<Log> logs;
    switch (op) {
      case KVM_SCHED_ALLOCATE: logs.push_back(h->s.allocate(ids[0], size)); break;
      case KVM_SCHED_DEPART: logs.push_back(h->s.depart(ids[0])); break;
      case KVM_SCHED_UPDATE: logs.push_back(h->s.update(ids[0])); break;
      case KVM_SCHED_HANDLE_GROWTH: h->s.handle_growth(std::vector<int64_t>(ids, ids + n_ids), logs); break;
      case KVM_SCHED_DUMP_CLASSES: {
        std::vector<std::pair<int64_t, int32_t>> v;
        h->s.sched_class.each([&](int64_t k, int32_t x) { v.push_back({k, x}); });
        std::sort(v.begin(), v.end());
        h->buf.clear();
        for (auto& p : v) emit(h->buf, KVM_REC_CLASS, p.first, p.second);
        *recs = h->buf.data();
        *n = (int64_t)h->buf.size() / 5;
        return KVM_OK;
      }
      default: raise(KVM_ERR_INVALID, "unknown scheduler op " + std::to_string(op));
    }
    h->buf.clear();
    emit_logs(h->buf, logs);
    *recs = h->buf.data();
    *n = (int64_t)h->buf.size() / 5;
    return KVM_OK;
  });
}

int kvm_sched_class_of(kvm_sched* h, int64_t item, int32_t* cls) {
  return guard([&] {
    if (!h || !cls) raise(KVM_ERR_INVALID, "NULL argument");
    const int32_t* p = h->s.sched_class.get(item);
    *cls = p ? *p : -1;
    return KVM_OK;
  });
}

int kvm_sched_priority(kvm_sched* h, int64_t src, int64_t dst, double* out) {
  return guard([&] {
    if (!h || !out) raise(KVM_ERR_INVALID, "NULL argument");
    *out = src == NONE ? h->s.alloc_prio(dst) : h->s.mig_prio(src, dst);
    return KVM_OK;
  });
}

}  // extern "C"
