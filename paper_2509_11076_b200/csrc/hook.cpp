// hook.cpp -- the profiler hook at operator dispatch in C++ (Chameleon hooks the
// framework's operator dispatch; matching must not make dispatch host-bound; Table 1,
// Lightweight mode +0.9% per iteration).  A PyTorch extension, separate from libchm
// (the C ABI carries no torch types): a boxed dispatcher fallback on a mode key that the runtime
// includes in the thread-local dispatch key set for the duration of a step (autograd's engine
// carries the thread-local state into its worker threads, so backward ops are seen too).  It
// sits above autograd, so it sees the ops the program calls (aten::linear, the backward
// formulas' aten::mm ...) with their real inputs and outputs; nested ops are excluded while one
// runs.  Per op it does what runtime.py's TorchDispatchMode did in Python:
//   Lightweight (no policy, nothing to record): token + phase appended to a buffer, handed to
//     chm_record_tokens once per step;
//   Detailed / with a policy: the op's record -- token, phase, the storages it reads and the
//     ones it creates (identity = storage address, App. A), in Detailed steps the storages freed
//     since (weak references) and the allocator's bytes in use -- is sent to
//     chm_record_op when the next op arrives (so frees between two ops and autograd's pack
//     hooks of the op come first); the executor's actions for it go to the Python runtime
//     (runtime.py _actions) only when there are any.
// OOM inside an op (Algo. 3): the runtime's callback makes room and the op is
// retried from a copy of its arguments.
// libchm's entry points come as addresses from the loaded library (one copy of the library in
// the process: the one chm.py loaded).
#include <ATen/core/dispatch/Dispatcher.h>
#include <ATen/core/ivalue.h>
#include <c10/core/impl/LocalDispatchKeySet.h>
#include <ATen/ops/empty.h>
#include <c10/cuda/CUDACachingAllocator.h>
#include <c10/cuda/CUDAStream.h>
#include <c10/util/Exception.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>
#include <torch/csrc/utils/pybind.h>  // at::Tensor <-> torch.Tensor casters
#include <torch/csrc/autograd/graph_task.h>
#include <torch/library.h>

#include <chrono>
#include <cstdint>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "chm.h"

namespace py = pybind11;

namespace {

constexpr c10::DispatchKey kKey = c10::DispatchKey::TESTING_ONLY_GenericMode;

using record_op_fn = chm_status (*)(chm_ctx *, const chm_op_record *, chm_actions *);
using tokenize_fn = chm_status (*)(chm_ctx *, const char *, int32_t *);
using record_tokens_fn = chm_status (*)(chm_ctx *, const int32_t *, const uint8_t *, uint32_t);
using last_error_fn = const char *(*)();
using issue_out_fn = chm_status (*)(chm_ctx *, cudaStream_t, cudaStream_t, uint32_t, uint64_t *);
using issue_in_fn = chm_status (*)(chm_ctx *, const uint64_t *, cudaStream_t, cudaStream_t, uint32_t, uint64_t *);
using item_wait_fn = chm_status (*)(chm_ctx *, uint32_t, int32_t, cudaStream_t);

struct Hook {
  chm_ctx *ctx = nullptr;       // the runtime whose step is running (attach .. detach)
  chm_ctx *last_ctx = nullptr;  // whose tokens the cache holds
  record_op_fn record_op = nullptr;
  tokenize_fn tokenize = nullptr;
  record_tokens_fn record_tokens = nullptr;
  last_error_fn last_error = nullptr;
  issue_out_fn issue_out = nullptr;
  issue_in_fn issue_in = nullptr;
  item_wait_fn item_wait = nullptr;
  cudaStream_t s_out = nullptr, s_in = nullptr;  // the runtime's swap streams
  uint32_t swap_flags = 0;
  std::unordered_map<uint32_t, chm_swap_desc> item_desc;  // policy item -> its swap-out descriptor
  int64_t n_swap_out = 0, n_swap_in = 0;
  std::vector<uint64_t> in_ptrs;
  int device = -1;  // CUDA device of the tracked tensors; -1: CPU tensors (host-only runtime)
  std::unordered_map<const void *, int32_t> tokens;  // operator schema -> token
  // step mode
  bool light = true, detailed = false, actions = false, oom = false;
  // per step
  std::vector<int32_t> tok;
  std::vector<uint8_t> ph;
  bool bwd_seen = false;
  uint8_t last_phase = CHM_FWD;
  int64_t n_ops = 0, n_actions = 0, n_oom_retries = 0;
  bool has_pending = false;
  int32_t p_tok = 0;
  uint8_t p_phase = 0;
  int64_t p_live = -1;
  std::vector<chm_tensor_ref> p_in, p_out;
  std::vector<uint64_t> freed;
  std::unordered_set<uint64_t> produced;
  std::unordered_set<uint64_t> statics;  // read before any op of the step created them
  // with OOM handling: weak references to the storages completed ops created, so a passive swap
  // only takes a storage that is still the one the executor recorded at that address
  std::unordered_map<uint64_t, c10::weak_intrusive_ptr<c10::StorageImpl>> live;
  std::unordered_map<uint64_t, c10::weak_intrusive_ptr<c10::StorageImpl>> weak;
  chm_actions act{};
  py::object on_actions, on_oom, on_release, on_swap_in;
  bool timing = false;      // measure the hook's own time per op (excluding the op itself)
  int64_t self_ns = 0, callback_ns = 0;
  std::string error;  // first failure inside a step (raised by end_step)
};

int64_t now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

Hook &H() {
  static Hook h;
  return h;
}

uint8_t dtype_code(c10::ScalarType t) {  // runtime.py _DTYPE_CODE
  switch (t) {
    case c10::ScalarType::Float: return 0;
    case c10::ScalarType::Half: return 1;
    case c10::ScalarType::BFloat16: return 2;
    case c10::ScalarType::Long: return 3;
    case c10::ScalarType::Int: return 4;
    case c10::ScalarType::Byte: return 5;
    case c10::ScalarType::Bool: return 6;
    case c10::ScalarType::Char: return 7;
    case c10::ScalarType::Double: return 8;
    case c10::ScalarType::Short: return 9;
    default: return 15;
  }
}

int32_t token_of(Hook &h, const c10::OperatorHandle &op) {
  const void *key = &op.schema();
  auto it = h.tokens.find(key);
  if (it != h.tokens.end()) return it->second;
  const auto &nm = op.operator_name();
  std::string s = nm.name;
  if (!nm.overload_name.empty()) s += "." + nm.overload_name;
  int32_t t = 0;
  if (h.tokenize(h.ctx, s.c_str(), &t) != CHM_OK) t = 1;
  h.tokens.emplace(key, t);
  return t;
}

uint8_t phase_now(Hook &h) {
  uint8_t ph;
  if (torch::autograd::get_current_graph_task_id() != -1) {
    h.bwd_seen = true;
    ph = CHM_BWD;
  } else {
    ph = h.bwd_seen ? CHM_OPT : CHM_FWD;
  }
  if (ph < h.last_phase) ph = h.last_phase;  // FWD* BWD* OPT* (runtime.py _stage)
  h.last_phase = ph;
  return ph;
}

bool tracked(const Hook &h, const at::Tensor &t) {
  if (!t.defined() || t.is_sparse() || !t.has_storage()) return false;
  const c10::Device d = t.device();
  return h.device < 0 ? d.is_cpu() : (d.is_cuda() && d.index() == h.device);
}

template <class F>
void for_each_tensor(const c10::IValue &v, F &&f) {
  if (v.isTensor()) {
    f(v.toTensor());
  } else if (v.isTensorList()) {
    for (const at::Tensor &t : v.toTensorVector()) f(t);
  } else if (v.isList()) {
    for (const c10::IValue &x : v.toListRef()) for_each_tensor(x, f);
  } else if (v.isTuple()) {
    for (const c10::IValue &x : v.toTupleRef().elements()) for_each_tensor(x, f);
  }
}

// the tracked storages among the values, deduplicated: (address, block bytes, dtype code)
void collect(const Hook &h, const c10::IValue &v, std::vector<chm_tensor_ref> &out) {
  for_each_tensor(v, [&](const at::Tensor &t) {
    if (!tracked(h, t)) return;
    const c10::Storage &st = t.storage();
    const uint64_t p = reinterpret_cast<uint64_t>(st.data());
    const int64_t nb = int64_t(st.nbytes());
    if (nb <= 0 || p == 0) return;
    for (const auto &r : out)
      if (r.id == p) return;
    out.push_back(chm_tensor_ref{p, nb, dtype_code(t.scalar_type())});
  });
}

void fail(Hook &h, const std::string &msg) {
  if (h.error.empty()) h.error = msg;
}

// sends the pending op's record (with the frees since it ran) and hands its actions over
void flush(Hook &h) {
  if (!h.has_pending) return;
  h.has_pending = false;
  h.freed.clear();
  if (h.detailed && !h.weak.empty()) {
    for (auto it = h.weak.begin(); it != h.weak.end();) {
      if (it->second.expired()) {
        h.freed.push_back(it->first);
        it = h.weak.erase(it);
      } else {
        ++it;
      }
    }
  }
  chm_op_record r{};
  r.token = h.p_tok;
  r.phase = h.p_phase;
  r.n_in = uint32_t(h.p_in.size());
  r.n_out = uint32_t(h.p_out.size());
  r.n_free = uint32_t(h.freed.size());
  r.in = h.p_in.data();
  r.out = h.p_out.data();
  r.freed = h.freed.data();
  r.live_bytes = h.p_live;
  if (h.record_op(h.ctx, &r, &h.act) != CHM_OK) {
    fail(h, std::string("chm_record_op: ") + (h.last_error ? h.last_error() : ""));
    return;
  }
  h.n_ops++;
  const chm_actions &a = h.act;
  if (!h.actions || !(a.n_swap_out || a.n_release || a.n_swap_in || a.n_wait)) return;
  h.n_actions++;
  if (h.device < 0) {  // host-only runtime: the Python executor glue does everything
    const int64_t t0 = h.timing ? now_ns() : 0;
    {
      py::gil_scoped_acquire gil;
      h.on_actions(reinterpret_cast<uintptr_t>(&h.act));
    }
    if (h.timing) h.callback_ns += now_ns() - t0;
    return;
  }
  // after op i (reading R-exec): swap-outs of the items matched at i, stream-ordered releases,
  // swap-ins of s_t = i + 1 into fresh blocks, waits for b_t = i + 1 -- in that order; the
  // releases and the new blocks' owners are the Python runtime's (autograd's boxes)
  cudaStream_t comp = c10::cuda::getCurrentCUDAStream(c10::DeviceIndex(h.device)).stream();
  auto check = [&](chm_status st, const char *what) {
    if (st != CHM_OK) fail(h, std::string(what) + ": " + (h.last_error ? h.last_error() : ""));
    return st == CHM_OK;
  };
  if (a.n_swap_out) {
    for (uint32_t j = 0; j < a.n_swap_out; j++) h.item_desc[a.swap_out_item[j]] = a.swap_out[j];
    uint64_t b = 0;
    if (!check(h.issue_out(h.ctx, comp, h.s_out, h.swap_flags, &b), "chm_issue_swap_out")) return;
    h.n_swap_out += a.n_swap_out;
  }
  const int64_t t0 = h.timing ? now_ns() : 0;
  if (a.n_release) {
    py::gil_scoped_acquire gil;
    py::list rel;
    for (uint32_t j = 0; j < a.n_release; j++) {
      const uint32_t it = a.release_item[j];
      auto d = h.item_desc.find(it);
      if (d == h.item_desc.end()) {
        fail(h, "release of an item never swapped out");
        continue;
      }
      rel.append(py::make_tuple(it, d->second.dev, d->second.host_off, d->second.nbytes));
    }
    h.on_release(rel);
  }
  if (a.n_swap_in) {
    std::vector<at::Tensor> blocks;
    blocks.reserve(a.n_swap_in);
    h.in_ptrs.resize(a.n_swap_in);
    for (uint32_t j = 0; j < a.n_swap_in; j++) {
      blocks.push_back(at::empty({int64_t(a.swap_in[j].nbytes)},
                                 at::TensorOptions().dtype(at::kByte).device(at::kCUDA, c10::DeviceIndex(h.device))));
      h.in_ptrs[j] = reinterpret_cast<uint64_t>(blocks.back().data_ptr());
    }
    uint64_t b = 0;
    if (check(h.issue_in(h.ctx, h.in_ptrs.data(), comp, h.s_in, h.swap_flags, &b), "chm_issue_swap_in")) {
      h.n_swap_in += a.n_swap_in;
      py::gil_scoped_acquire gil;
      py::list got;
      for (uint32_t j = 0; j < a.n_swap_in; j++) got.append(py::make_tuple(a.swap_in_item[j], blocks[j]));
      h.on_swap_in(got);  // the runtime hands each block to its box (or waits and drops it)
    }
  }
  if (h.timing && (a.n_release || a.n_swap_in)) h.callback_ns += now_ns() - t0;
  for (uint32_t j = 0; j < a.n_wait; j++)  // before b_t: no block is read early (the unpack also waits)
    check(h.item_wait(h.ctx, a.wait_item[j], 1, comp), "chm_item_wait");
}

void redispatch(const c10::OperatorHandle &op, c10::DispatchKeySet ks, torch::jit::Stack *stack) {
  Hook &h = H();
  if (!h.timing) return op.redispatchBoxed(ks & c10::DispatchKeySet(c10::DispatchKeySet::FULL_AFTER, kKey), stack);
  const int64_t t0 = now_ns();
  op.redispatchBoxed(ks & c10::DispatchKeySet(c10::DispatchKeySet::FULL_AFTER, kKey), stack);
  h.self_ns -= now_ns() - t0;  // the op's own time is not the hook's
}

struct SelfTimer {  // the hook's time in one fallback call (the op's own time subtracted)
  Hook &h;
  int64_t t0;
  explicit SelfTimer(Hook &hh) : h(hh), t0(hh.timing ? now_ns() : 0) {}
  ~SelfTimer() {
    if (h.timing) h.self_ns += now_ns() - t0;
  }
};

void hook_fallback(const c10::OperatorHandle &op, c10::DispatchKeySet ks, torch::jit::Stack *stack) {
  c10::impl::ExcludeDispatchKeyGuard nested(kKey);  // the ops this one calls are not recorded
  Hook &h = H();
  if (!h.ctx) return redispatch(op, ks, stack);
  SelfTimer timer(h);
  if (h.light) {
    redispatch(op, ks, stack);
    h.tok.push_back(token_of(h, op));
    h.ph.push_back(phase_now(h));
    return;
  }
  flush(h);
  const size_t nargs = op.schema().arguments().size();
  std::vector<chm_tensor_ref> ins;
  for (size_t j = stack->size() - nargs; j < stack->size(); j++) collect(h, (*stack)[j], ins);
  for (const auto &i : ins)
    if (!h.produced.count(i.id)) h.statics.insert(i.id);  // weights, inputs: live before the step
  std::vector<c10::IValue> saved;
  if (h.oom) saved.assign(stack->end() - nargs, stack->end());
  for (;;) {
    try {
      redispatch(op, ks, stack);
      break;
    } catch (const c10::OutOfMemoryError &e) {  // Algo. 3: make room, then retry the op
      if (!h.oom) throw;
      bool retry = false;
      {
        py::gil_scoped_acquire gil;
        py::list busy;
        for (const auto &r : ins) busy.append(py::int_(r.id));
        retry = h.on_oom(std::string(e.what()), busy).cast<bool>();
      }
      if (!retry) throw;
      h.n_oom_retries++;
      stack->resize(stack->size() - std::min(stack->size(), nargs));  // whatever the failed call left
      stack->insert(stack->end(), saved.begin(), saved.end());
    }
  }
  const size_t nret = op.schema().returns().size();
  std::vector<chm_tensor_ref> outs_all, outs;
  for (size_t j = stack->size() - nret; j < stack->size(); j++) collect(h, (*stack)[j], outs_all);
  for (const auto &o : outs_all) {  // views and in-place outputs are uses, not new tensors
    bool is_in = false;
    for (const auto &i : ins) is_in = is_in || i.id == o.id;
    if (!is_in) outs.push_back(o);
  }
  h.p_live = -1;
  if (h.detailed) {
    if (h.device >= 0)
      h.p_live = int64_t(c10::cuda::CUDACachingAllocator::getDeviceStats(h.device)
                             .allocated_bytes[size_t(c10::CachingAllocator::StatType::AGGREGATE)]
                             .current);
    else
      h.p_live = 0;
    // weak references to the storages this op created: polled for frees at the next flush
    for (size_t j = stack->size() - nret; j < stack->size(); j++)
      for_each_tensor((*stack)[j], [&](const at::Tensor &t) {
        if (!tracked(h, t)) return;
        const uint64_t p = reinterpret_cast<uint64_t>(t.storage().data());
        for (const auto &o : outs)
          if (o.id == p) {
            h.weak.insert_or_assign(p, t.storage().getWeakStorageImpl());
            break;
          }
      });
  }
  for (const auto &o : outs) h.produced.insert(o.id);
  if (h.oom)
    for (size_t j = stack->size() - nret; j < stack->size(); j++)
      for_each_tensor((*stack)[j], [&](const at::Tensor &t) {
        if (!tracked(h, t)) return;
        const uint64_t p = reinterpret_cast<uint64_t>(t.storage().data());
        for (const auto &o : outs)
          if (o.id == p) {
            h.live.insert_or_assign(p, t.storage().getWeakStorageImpl());
            break;
          }
      });
  h.p_tok = token_of(h, op);
  h.p_phase = phase_now(h);
  h.p_in = std::move(ins);
  h.p_out = std::move(outs);
  h.has_pending = true;
}

}  // namespace

TORCH_LIBRARY_IMPL(_, TESTING_ONLY_GenericMode, m) {
  m.fallback(torch::CppFunction::makeFromBoxedFunction<&hook_fallback>());
}

PYBIND11_MODULE(TORCH_EXTENSION_NAME, m) {
  m.doc() = "Chameleon profiler hook at operator dispatch (C++), see csrc/hook.cpp";
  m.def("attach", [](uintptr_t ctx, uintptr_t record_op, uintptr_t tokenize, uintptr_t record_tokens,
                     uintptr_t last_error, int device, py::object on_actions, py::object on_oom,
                     uintptr_t issue_out, uintptr_t issue_in, uintptr_t item_wait, uintptr_t s_out, uintptr_t s_in,
                     uint32_t swap_flags, py::object on_release, py::object on_swap_in) {
    Hook &h = H();
    if (h.ctx && ctx && h.ctx != reinterpret_cast<chm_ctx *>(ctx))
      throw std::runtime_error("chm hook: another runtime's step is running in this process");
    if (reinterpret_cast<chm_ctx *>(ctx) != h.last_ctx) h.tokens.clear();  // tokens are per ctx
    h.ctx = reinterpret_cast<chm_ctx *>(ctx);
    h.last_ctx = h.ctx;
    h.record_op = reinterpret_cast<record_op_fn>(record_op);
    h.tokenize = reinterpret_cast<tokenize_fn>(tokenize);
    h.record_tokens = reinterpret_cast<record_tokens_fn>(record_tokens);
    h.last_error = reinterpret_cast<last_error_fn>(last_error);
    h.device = device;
    h.on_actions = std::move(on_actions);
    h.on_oom = std::move(on_oom);
    h.issue_out = reinterpret_cast<issue_out_fn>(issue_out);
    h.issue_in = reinterpret_cast<issue_in_fn>(issue_in);
    h.item_wait = reinterpret_cast<item_wait_fn>(item_wait);
    h.s_out = reinterpret_cast<cudaStream_t>(s_out);
    h.s_in = reinterpret_cast<cudaStream_t>(s_in);
    h.swap_flags = swap_flags;
    h.on_release = std::move(on_release);
    h.on_swap_in = std::move(on_swap_in);
  });
  m.def("detach", []() {
    Hook &h = H();
    c10::impl::tls_set_dispatch_key_included(kKey, false);
    h.ctx = nullptr;
    h.on_actions = py::none();
    h.on_oom = py::none();
    h.on_release = py::none();
    h.on_swap_in = py::none();
    h.weak.clear();
  });
  m.def("forget", [](uintptr_t ctx) {  // a ctx about to be destroyed: its address may be reused
    Hook &h = H();
    if (h.last_ctx == reinterpret_cast<chm_ctx *>(ctx)) {
      h.last_ctx = nullptr;
      h.tokens.clear();
    }
  });
  m.def("set_timing", [](bool on) { H().timing = on; });
  // (hook self time incl. callbacks, Python callback time) of the last step, ns
  m.def("timing", []() { return py::make_tuple(H().self_ns, H().callback_ns); });
  m.def("begin_step", [](bool light, bool detailed, bool actions, bool oom) {
    Hook &h = H();
    h.self_ns = h.callback_ns = 0;
    h.light = light;
    h.detailed = detailed;
    h.actions = actions;
    h.oom = oom;
    h.tok.clear();
    h.ph.clear();
    h.bwd_seen = false;
    h.last_phase = CHM_FWD;
    h.n_ops = h.n_actions = h.n_oom_retries = 0;
    h.n_swap_out = h.n_swap_in = 0;
    h.item_desc.clear();
    h.has_pending = false;
    h.produced.clear();
    h.statics.clear();
    h.live.clear();
    h.weak.clear();
    h.error.clear();
  });
  // the calling thread's dispatch key set (autograd copies it into its worker threads)
  m.def("enable", [](bool on) { c10::impl::tls_set_dispatch_key_included(kKey, on); });
  m.def("enabled", []() { return c10::impl::tls_is_dispatch_key_included(kKey); });
  m.def("end_step", []() {
    Hook &h = H();
    c10::impl::ExcludeDispatchKeyGuard nested(kKey);
    if (h.light) {
      if (!h.tok.empty() && h.record_tokens(h.ctx, h.tok.data(), h.ph.data(), uint32_t(h.tok.size())) != CHM_OK)
        fail(h, std::string("chm_record_tokens: ") + (h.last_error ? h.last_error() : ""));
      h.n_ops = int64_t(h.tok.size());
    } else {
      flush(h);
    }
    h.weak.clear();
    h.live.clear();
    if (!h.error.empty()) {
      std::string e = h.error;
      h.error.clear();
      throw std::runtime_error(e);
    }
    return py::make_tuple(h.n_ops, h.n_actions, h.n_oom_retries, h.n_swap_out, h.n_swap_in);
  });
  m.def("abort_step", []() {
    Hook &h = H();
    h.has_pending = false;
    h.tok.clear();
    h.ph.clear();
    h.weak.clear();
    h.produced.clear();
    h.statics.clear();
    h.live.clear();
    h.error.clear();
  });
  m.def("produced", [](uint64_t p) { return H().produced.count(p) != 0; });
  // (OOM handling) p is a storage a completed op of this step created, still alive: the
  // executor's record at that address is this storage (not a reused address)
  m.def("produced_live", [](uint64_t p) {
    const auto &L = H().live;
    auto it = L.find(p);
    return it != L.end() && !it->second.expired();
  });
  // autograd's pack hook of an op runs inside it, before the op's outputs are recorded: a
  // storage is the step's own unless an op read it before any op of the step created it
  m.def("is_static", [](uint64_t p) { return H().statics.count(p) != 0; });
}
