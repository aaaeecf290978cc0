// tk_texcache.cu -- the pooled texture arrays declared in tk_tex.cuh.
#include <algorithm>
#include <list>
#include <memory>
#include <mutex>

#include "tk_common.cuh"
#include "tk_tex.cuh"

namespace tk {

namespace {

struct Slot {
  int dev = 0;
  int w = 0, h = 0, layers = 0;
  TexKind kind = TexKind::kLayeredPoint;
  cudaArray_t arr = nullptr;
  cudaTextureObject_t tex = 0;
  cudaEvent_t done = nullptr;  // recorded after the last consumer
  bool busy = false;
  bool used = false;
  unsigned long long last_use = 0;
  size_t bytes() const { return (size_t)w * h * std::max(layers, 1) * sizeof(float); }
  void destroy() {
    if (tex) cudaDestroyTextureObject(tex);
    if (arr) cudaFreeArray(arr);
    if (done) cudaEventDestroy(done);
    tex = 0;
    arr = nullptr;
    done = nullptr;
  }
};

std::mutex g_mu;
std::list<std::unique_ptr<Slot>> g_slots;
unsigned long long g_clock = 0;
size_t g_limit = (size_t)24 << 30;  // cached bytes kept across calls

size_t cached_bytes() {
  size_t s = 0;
  for (auto &p : g_slots) s += p->bytes();
  return s;
}

void evict_idle_locked(size_t need) {
  while (cached_bytes() + need > g_limit) {
    Slot *victim = nullptr;
    for (auto &p : g_slots)
      if (!p->busy && (!victim || p->last_use < victim->last_use)) victim = p.get();
    if (!victim) return;
    if (victim->done) cudaEventSynchronize(victim->done);
    victim->destroy();
    g_slots.remove_if([victim](const std::unique_ptr<Slot> &p) { return p.get() == victim; });
  }
}

cudaError_t create(Slot &s) {
  cudaChannelFormatDesc fmt = cudaCreateChannelDesc<float>();
  cudaError_t e;
  if (s.kind == TexKind::kVolumeLinear) {
    e = cudaMalloc3DArray(&s.arr, &fmt, make_cudaExtent(s.w, s.h, s.layers), 0);
  } else {
    e = cudaMalloc3DArray(&s.arr, &fmt, make_cudaExtent(s.w, s.h, s.layers), cudaArrayLayered);
  }
  if (e != cudaSuccess) return e;
  cudaResourceDesc res = {};
  res.resType = cudaResourceTypeArray;
  res.res.array.array = s.arr;
  cudaTextureDesc td = {};
  for (int i = 0; i < 3; ++i) td.addressMode[i] = cudaAddressModeBorder;
  td.borderColor[0] = td.borderColor[1] = td.borderColor[2] = td.borderColor[3] = 0.f;
  td.filterMode = s.kind == TexKind::kLayeredPoint ? cudaFilterModePoint : cudaFilterModeLinear;
  td.readMode = cudaReadModeElementType;
  td.normalizedCoords = 0;
  e = cudaCreateTextureObject(&s.tex, &res, &td, nullptr);
  if (e != cudaSuccess) return e;
  return cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming);
}

}  // namespace

cudaError_t tex_acquire(const float *src, int w, int h, int layers, TexKind kind, cudaStream_t st,
                        TexLease &out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  Slot *slot = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_mu);
    for (auto &p : g_slots) {
      if (!p->busy && p->dev == dev && p->w == w && p->h == h && p->layers == layers && p->kind == kind) {
        slot = p.get();
        break;
      }
    }
    if (!slot) {
      auto s = std::make_unique<Slot>();
      s->dev = dev;
      s->w = w;
      s->h = h;
      s->layers = layers;
      s->kind = kind;
      evict_idle_locked(s->bytes());
      e = create(*s);
      if (e != cudaSuccess) {
        s->destroy();
        return e;
      }
      slot = s.get();
      g_slots.push_back(std::move(s));
    }
    slot->busy = true;
    slot->last_use = ++g_clock;
  }
  if (slot->used) {  // order our overwrite after the previous consumer
    e = cudaStreamWaitEvent(st, slot->done, 0);
    if (e != cudaSuccess) return e;
  }
  cudaMemcpy3DParms cp = {};
  cp.srcPtr = make_cudaPitchedPtr(const_cast<float *>(src), (size_t)w * sizeof(float), w, h);
  cp.dstArray = slot->arr;
  cp.extent = make_cudaExtent(w, h, layers);
  cp.kind = cudaMemcpyDeviceToDevice;
  e = cudaMemcpy3DAsync(&cp, st);
  if (e != cudaSuccess) return e;
  out.tex = slot->tex;
  out.slot = slot;
  return cudaSuccess;
}

void tex_release(TexLease &lease, cudaStream_t st) {
  Slot *slot = reinterpret_cast<Slot *>(lease.slot);
  if (!slot) return;
  cudaEventRecord(slot->done, st);
  std::lock_guard<std::mutex> lock(g_mu);
  slot->used = true;
  slot->busy = false;
  lease.slot = nullptr;
  lease.tex = 0;
}

}  // namespace tk

extern "C" {

// Free every idle pooled texture array (they are re-created on demand).
int tk_release_cached_memory(void) {
  tk::clear_error();
  std::lock_guard<std::mutex> lock(tk::g_mu);
  for (auto it = tk::g_slots.begin(); it != tk::g_slots.end();) {
    if (!(*it)->busy) {
      if ((*it)->done) cudaEventSynchronize((*it)->done);
      (*it)->destroy();
      it = tk::g_slots.erase(it);
    } else {
      ++it;
    }
  }
  return TK_OK;
}

// Bytes currently held by the texture-array pool.
unsigned long long tk_cached_bytes(void) {
  std::lock_guard<std::mutex> lock(tk::g_mu);
  return tk::cached_bytes();
}

}  // extern "C"
