// api.cu — extern "C" entry points of libsmat.so (see include/smat.h).
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "plan.cuh"

struct smat_plan {
  smat::Plan* p = nullptr;
  // staging buffers of smat_apply_host (grown on demand, guarded by mu)
  std::mutex mu;
  cudaStream_t streams[3] = {nullptr, nullptr, nullptr};
  void* dx[3] = {nullptr, nullptr, nullptr};
  void* dy[3] = {nullptr, nullptr, nullptr};
  void* dw[3] = {nullptr, nullptr, nullptr};
  size_t bx = 0, by = 0, bw = 0;
};

namespace {
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

template <class F>
int guarded(F f) {
  try {
    f();
    return SMAT_OK;
  } catch (const smat::Error& e) {
    return fail(e.code, e.what());
  } catch (const std::bad_alloc&) {
    return fail(SMAT_OOM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(SMAT_BAD_ARG, e.what());
  }
}

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) SMAT_CUDA(cudaSetDevice(d));
  }
  ~DeviceGuard() {
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != prev) cudaSetDevice(prev);
  }
};

size_t measure(const smat::Plan& p, int dir, int64_t ncols, int64_t* launches, int64_t ldx = 0, int64_t ldy = 0,
               int layout = SMAT_ROW_MAJOR) {
  smat::Ctx c;
  c.device = p.device;
  c.dt = p.dt;
  c.measure = true;
  static char dummy;
  smat::run_plan(p, c, dir, &dummy, p.dt, ldx, &dummy, ldy, ncols, layout);
  if (launches) *launches = c.launches;
  size_t peak = c.peak;
  if (smat::dt_complex(p.dt)) {
    // a real input to a complex plan may need a promoted copy first
    smat::Ctx r;
    r.device = p.device;
    r.dt = p.dt;
    r.measure = true;
    smat::run_plan(p, r, dir, &dummy, smat::dt_real_of(p.dt), ldx, &dummy, ldy, ncols, layout);
    if (r.peak > peak) peak = r.peak;
  }
  return peak;
}

int check_apply_args(const smat::Plan& p, int direction, int x_dtype, int64_t ncols, int layout) {
  if (direction != 0 && direction != 1) return fail(SMAT_BAD_ARG, "direction must be 0 or 1");
  if (ncols < 1) return fail(SMAT_BAD_SHAPE, "ncols must be >= 1");
  if (layout != SMAT_ROW_MAJOR && layout != SMAT_COL_MAJOR) return fail(SMAT_BAD_ARG, "unknown layout");
  if (x_dtype != p.dt && !(smat::dt_complex(p.dt) && x_dtype == smat::dt_real_of(p.dt)))
    return fail(SMAT_BAD_DTYPE, "input dtype does not match the plan dtype");
  return SMAT_OK;
}
}  // namespace

namespace smat {
void set_last_error(const std::string& m) { g_err = m; }
double probe_peak_tflops(int kind, int device);  // probe.cu
}  // namespace smat

extern "C" {

int smat_abi_version(void) { return SMAT_ABI_VERSION; }

const char* smat_last_error(void) { return g_err.c_str(); }

int smat_plan_build(const smat_node* nodes, int32_t n_nodes, const int32_t* children, int32_t n_children,
                    int32_t root, int32_t dtype, int32_t device, smat_plan** out) {
  if (!nodes || !out || n_nodes <= 0) return fail(SMAT_BAD_ARG, "smat_plan_build: null argument");
  *out = nullptr;
  return guarded([&] {
    DeviceGuard dg(device);
    auto* h = new smat_plan;
    try {
      h->p = smat::build_plan(nodes, n_nodes, children, n_children, root, dtype, device);
      // dry runs create the shared twiddle tables now, so that apply() never
      // allocates or synchronises (CUDA-graph capturable).
      measure(*h->p, 0, 1, nullptr);
      measure(*h->p, 1, 1, nullptr);
    } catch (...) {
      delete h->p;
      delete h;
      throw;
    }
    *out = h;
  });
}

int smat_workspace_bytes(const smat_plan* plan, int32_t direction, int64_t ncols, int64_t ldx, int64_t ldy,
                         int32_t layout, size_t* out_bytes) {
  if (!plan || !out_bytes) return fail(SMAT_BAD_ARG, "null argument");
  return guarded([&] {
    DeviceGuard dg(plan->p->device);
    *out_bytes = measure(*plan->p, direction, ncols, nullptr, ldx, ldy, layout);
  });
}

int smat_probe_peak(int32_t kind, int32_t device, double* tflops) {
  if (!tflops || kind < 0 || kind > 3) return fail(SMAT_BAD_ARG, "smat_probe_peak: bad argument");
  return guarded([&] { *tflops = smat::probe_peak_tflops(kind, device); });
}

int smat_plan_launches(const smat_plan* plan, int32_t direction, int64_t ncols, int64_t* out_launches) {
  if (!plan || !out_launches) return fail(SMAT_BAD_ARG, "null argument");
  return guarded([&] {
    DeviceGuard dg(plan->p->device);
    measure(*plan->p, direction, ncols, out_launches);
  });
}

int smat_plan_describe(const smat_plan* plan, char* buf, size_t buf_len) {
  if (!plan || !buf || !buf_len) return fail(SMAT_BAD_ARG, "null argument");
  std::string s = plan->p->root->describe();
  if (!plan->p->fused.empty()) s += " [fused: " + plan->p->fused + "]";
  std::strncpy(buf, s.c_str(), buf_len - 1);
  buf[buf_len - 1] = 0;
  return SMAT_OK;
}

int smat_plan_shape(const smat_plan* plan, int64_t* rows, int64_t* cols, int32_t* dtype) {
  if (!plan) return fail(SMAT_BAD_ARG, "null plan");
  if (rows) *rows = plan->p->rows;
  if (cols) *cols = plan->p->cols;
  if (dtype) *dtype = plan->p->dt;
  return SMAT_OK;
}

int smat_apply(const smat_plan* plan, int32_t direction, const void* x, int32_t x_dtype, int64_t ldx, void* y,
               int64_t ldy, int64_t ncols, int32_t layout, void* workspace, size_t workspace_bytes, void* stream) {
  if (!plan || !x || !y) return fail(SMAT_BAD_ARG, "smat_apply: null argument");
  const smat::Plan& p = *plan->p;
  if (int st = check_apply_args(p, direction, x_dtype, ncols, layout)) return st;
  return guarded([&] {
    DeviceGuard dg(p.device);
    smat::Ctx c;
    c.device = p.device;
    c.dt = p.dt;
    c.stream = (cudaStream_t)stream;
    c.ws = (char*)workspace;
    c.ws_size = workspace ? workspace_bytes : 0;
    smat::run_plan(p, c, direction, x, x_dtype, ldx, y, ldy, ncols, layout);
  });
}

int smat_apply_profiled(const smat_plan* plan, int32_t direction, const void* x, int32_t x_dtype, void* y,
                        int64_t ncols, void* workspace, size_t workspace_bytes, void* stream, float* launch_ms,
                        int32_t max_launches, int32_t* n_launches, char* labels, size_t labels_len) {
  if (!plan || !x || !y || !launch_ms || !n_launches) return fail(SMAT_BAD_ARG, "smat_apply_profiled: null argument");
  if (direction != 0 && direction != 1) return fail(SMAT_BAD_ARG, "direction must be 0 or 1");
  const smat::Plan& p = *plan->p;
  if (x_dtype != p.dt && !(smat::dt_complex(p.dt) && x_dtype == smat::dt_real_of(p.dt)))
    return fail(SMAT_BAD_DTYPE, "input dtype does not match the plan dtype");
  std::vector<std::pair<std::string, cudaEvent_t>> ev;
  int st = guarded([&] {
    DeviceGuard dg(p.device);
    smat::Ctx c;
    c.device = p.device;
    c.dt = p.dt;
    c.stream = (cudaStream_t)stream;
    c.ws = (char*)workspace;
    c.ws_size = workspace ? workspace_bytes : 0;
    c.prof = &ev;
    smat::run_plan(p, c, direction, x, x_dtype, 0, y, 0, ncols, SMAT_ROW_MAJOR);
    c.note("end");
    SMAT_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    std::string lab;
    int n = 0;
    for (size_t i = 0; i + 1 < ev.size() && n < max_launches; ++i, ++n) {
      float ms = 0.f;
      SMAT_CUDA(cudaEventElapsedTime(&ms, ev[i].second, ev[i + 1].second));
      launch_ms[n] = ms;
      lab += ev[i].first + "\n";
    }
    *n_launches = n;
    if (labels && labels_len) {
      std::strncpy(labels, lab.c_str(), labels_len - 1);
      labels[labels_len - 1] = 0;
    }
  });
  for (auto& e : ev) cudaEventDestroy(e.second);
  return st;
}

int smat_apply_host(const smat_plan* plan_c, int32_t direction, const void* x_host, int32_t x_dtype, int64_t ldx,
                    void* y_host, int64_t ldy, int64_t ncols, int32_t layout, int32_t chunk_cols) {
  smat_plan* plan = const_cast<smat_plan*>(plan_c);
  if (!plan || !x_host || !y_host) return fail(SMAT_BAD_ARG, "smat_apply_host: null argument");
  const smat::Plan& p = *plan->p;
  if (int st = check_apply_args(p, direction, x_dtype, ncols, layout)) return st;
  const bool adj = direction == 1;
  const int64_t nin = adj ? p.rows : p.cols, nout = adj ? p.cols : p.rows;
  const bool col = layout == SMAT_COL_MAJOR;
  if (ldx <= 0) ldx = col ? nin : ncols;
  if (ldy <= 0) ldy = col ? nout : ncols;
  if (ldx < (col ? nin : ncols) || ldy < (col ? nout : ncols))
    return fail(SMAT_BAD_ARG, "leading dimension smaller than the block");
  return guarded([&] {
    std::lock_guard<std::mutex> lk(plan->mu);
    DeviceGuard dg(p.device);
    const size_t ex = smat::dt_size(x_dtype), ey = smat::dt_size(p.dt);
    int64_t cc = chunk_cols > 0 ? chunk_cols : ncols;
    if (cc > ncols) cc = ncols;
    const int64_t nchunks = (ncols + cc - 1) / cc;
    const int S = nchunks >= 3 ? 3 : int(nchunks);
    const size_t need_x = size_t(nin) * cc * ex, need_y = size_t(nout) * cc * ey;
    // device blocks are dense in the caller's layout (column-major chunks:
    // ld = rows); the chunk loop below moves them with pitched copies
    const size_t need_w = measure(p, direction, cc, nullptr, 0, 0, layout);
    auto grow = [&](void** arr, size_t& have, size_t need) {
      if (need <= have) return;
      have = 0;  // (committed only once every buffer is allocated)
      for (int i = 0; i < 3; ++i)
        if (arr[i]) {
          cudaFree(arr[i]);
          arr[i] = nullptr;
        }
      for (int i = 0; i < 3; ++i) SMAT_CUDA(cudaMalloc(&arr[i], need ? need : 1));
      have = need;
    };
    grow(plan->dx, plan->bx, need_x);
    grow(plan->dy, plan->by, need_y);
    grow(plan->dw, plan->bw, need_w);
    for (int i = 0; i < 3; ++i)
      if (!plan->streams[i]) SMAT_CUDA(cudaStreamCreateWithFlags(&plan->streams[i], cudaStreamNonBlocking));
    try {
      for (int64_t k = 0; k < nchunks; ++k) {
        const int s = int(k % S);
        const int64_t c0 = k * cc, w = std::min<int64_t>(cc, ncols - c0);
        cudaStream_t st = plan->streams[s];
        if (col) {  // w contiguous columns of nin elements, ldx apart
          SMAT_CUDA(cudaMemcpy2DAsync(plan->dx[s], size_t(nin) * ex, (const char*)x_host + size_t(c0) * ldx * ex,
                                      size_t(ldx) * ex, size_t(nin) * ex, size_t(w), cudaMemcpyHostToDevice, st));
        } else if (w == ncols && ldx == ncols) {  // whole dense block: one contiguous DMA at full link bandwidth
          SMAT_CUDA(cudaMemcpyAsync(plan->dx[s], x_host, size_t(nin) * ncols * ex, cudaMemcpyHostToDevice, st));
        } else {  // column chunk of a row-major block: pitched copy
          SMAT_CUDA(cudaMemcpy2DAsync(plan->dx[s], size_t(w) * ex, (const char*)x_host + size_t(c0) * ex,
                                      size_t(ldx) * ex, size_t(w) * ex, size_t(nin), cudaMemcpyHostToDevice, st));
        }
        smat::Ctx c;
        c.device = p.device;
        c.dt = p.dt;
        c.stream = st;
        c.ws = (char*)plan->dw[s];
        c.ws_size = plan->bw;
        smat::run_plan(p, c, direction, plan->dx[s], x_dtype, 0, plan->dy[s], 0, w, layout);
        if (col) {
          SMAT_CUDA(cudaMemcpy2DAsync((char*)y_host + size_t(c0) * ldy * ey, size_t(ldy) * ey, plan->dy[s],
                                      size_t(nout) * ey, size_t(nout) * ey, size_t(w), cudaMemcpyDeviceToHost, st));
        } else if (w == ncols && ldy == ncols) {
          SMAT_CUDA(cudaMemcpyAsync(y_host, plan->dy[s], size_t(nout) * ncols * ey, cudaMemcpyDeviceToHost, st));
        } else {
          SMAT_CUDA(cudaMemcpy2DAsync((char*)y_host + size_t(c0) * ey, size_t(ldy) * ey, plan->dy[s],
                                      size_t(w) * ey, size_t(w) * ey, size_t(nout), cudaMemcpyDeviceToHost, st));
        }
      }
    } catch (...) {
      // the caller frees the host buffers once this returns: drain every
      // copy already queued first
      for (int i = 0; i < S; ++i) cudaStreamSynchronize(plan->streams[i]);
      throw;
    }
    for (int i = 0; i < S; ++i) SMAT_CUDA(cudaStreamSynchronize(plan->streams[i]));
  });
}

void smat_plan_free(smat_plan* plan) {
  if (!plan) return;
  {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(plan->p->device);
    for (int i = 0; i < 3; ++i) {
      if (plan->streams[i]) cudaStreamSynchronize(plan->streams[i]);
      if (plan->dx[i]) cudaFree(plan->dx[i]);
      if (plan->dy[i]) cudaFree(plan->dy[i]);
      if (plan->dw[i]) cudaFree(plan->dw[i]);
      if (plan->streams[i]) cudaStreamDestroy(plan->streams[i]);
    }
    delete plan->p;
    cudaSetDevice(prev);
  }
  delete plan;
}

}  // extern "C"
