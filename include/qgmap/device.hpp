// qgmap/device.hpp -- C++ side of the C ABI (include/qgm_c.h): device context,
// RAII handles and the translation of status codes back into the reference's
// exception types (input_error, seq.hpp:13-16; std::logic_error,
// parallel.hpp:176,181). Link with libqgm_b200.so.
#pragma once

#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>

#include "qgm_c.h"
#include "qgmap/seq.hpp"

namespace qgmap::device {

struct cuda_error : std::runtime_error {
  explicit cuda_error(const std::string& w) : std::runtime_error(w) {}
};

inline void check(int rc, const qgm_ctx* ctx) {
  if (rc == QGM_OK) return;
  const std::string msg = qgm_last_error(ctx);
  if (rc == QGM_ERR_INPUT) throw input_error(msg);
  if (rc == QGM_ERR_INTERNAL) throw std::logic_error(msg);
  throw cuda_error(msg);
}

// One CUDA device + stream. Every device object keeps its context alive.
class Context {
 public:
  explicit Context(int device = 0) {
    qgm_ctx* c = nullptr;
    const int rc = qgm_ctx_create(device, &c);
    if (rc != QGM_OK) throw cuda_error("qgm_ctx_create failed for device " + std::to_string(device));
    ctx_.reset(c, qgm_ctx_destroy);
  }
  qgm_ctx* get() const { return ctx_.get(); }
  void check(int rc) const { device::check(rc, ctx_.get()); }
  void synchronize() const { check(qgm_ctx_synchronize(ctx_.get())); }

  // Process-wide default context on device 0 (the reference API has no
  // context argument; threads= parameters are accepted and ignored).
  static std::shared_ptr<Context> default_context() {
    static std::mutex m;
    static std::shared_ptr<Context> d;
    std::lock_guard<std::mutex> lk(m);
    if (!d) d = std::make_shared<Context>(0);
    return d;
  }

 private:
  std::shared_ptr<qgm_ctx> ctx_;
};

// Owning handle that also pins its context (objects must die before it).
template <class T, void (*Destroy)(T*)>
struct Handle {
  std::shared_ptr<Context> ctx;
  std::shared_ptr<T> h;
  Handle() = default;
  Handle(std::shared_ptr<Context> c, T* raw) : ctx(std::move(c)) {
    auto keep = ctx;
    h = std::shared_ptr<T>(raw, [keep](T* p) { Destroy(p); });
  }
  T* get() const { return h.get(); }
  explicit operator bool() const { return bool(h); }
};

using ReadsHandle = Handle<qgm_reads, qgm_reads_destroy>;
using IndexHandle = Handle<qgm_index, qgm_index_destroy>;
using RefHandle = Handle<qgm_ref, qgm_ref_destroy>;

// Upload a PackedReadText (seq.hpp:98-115) to the device.
inline ReadsHandle upload_reads(const PackedReadText& text, std::shared_ptr<Context> ctx = Context::default_context()) {
  const auto words = text.pack();
  qgm_reads* r = nullptr;
  ctx->check(qgm_reads_upload(ctx->get(), words.data(), text.read_lengths.data(), text.read_count, text.stride, &r));
  return ReadsHandle(ctx, r);
}

}  // namespace qgmap::device
