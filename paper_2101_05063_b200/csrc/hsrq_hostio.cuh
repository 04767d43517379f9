// hsrq_hostio.cuh -- host-side I/O of the drop-in API (included by
// hsrq_kernels.cu): what hsrq3in / dhsrq3in / chsrq3in (inviter.py:155-254)
// pay around the solve when called with numpy arrays.
//
//   hsrq_h_upload        the caller's H (pageable numpy, C- or F-order) ->
//                        the device's column-major, even-ld H, through a
//                        pinned staging ring filled by host worker threads
//                        (one pageable cudaMemcpy runs at ~11 GB/s on this
//                        pool, pinned copies at ~55 GB/s); a C-order H lands
//                        as row blocks and is transposed on the device.
//                        Then one kernel computes what HessenbergMatrix
//                        checks and caches (core.py:60-98): the structure
//                        (nonzeros below the subdiagonal), unreducedness,
//                        and the infinity norm EXACTLY as the reference's
//                        np.max(np.sum(np.abs(F-order data), axis=1)) --
//                        a left-to-right sum per row, which is the order
//                        numpy reduces a Fortran-ordered array in.
//   hsrq_pack_download   the solve's column layout (X rows = columns, complex
//                        shifts as re/im pairs, any shift order) -> the
//                        caller's (n, m) C-order complex128 (or float64)
//                        vectors in caller order, conjugated where asked
//                        (chsrq3in's Im < 0 inputs, inviter.py:174-182):
//                        a tiled transpose kernel packs row blocks on the
//                        device, the blocks stream back through the pinned
//                        ring and worker threads copy them into the numpy
//                        result.
#include <condition_variable>
#include <functional>
#include <thread>

namespace hostio {

constexpr int NSLOT = 4;
constexpr size_t SLOT_BYTES = size_t(32) << 20;  // 32 MiB per staging slot

// Persistent worker threads for the host memcpys (pageable <-> pinned).
class Pool {
 public:
  explicit Pool(int n) {
    for (int i = 0; i < n; i++) th_.emplace_back([this] { run(); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> l(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return (int)th_.size(); }
  // run f(0..parts-1) on the workers, return when all are done
  void parallel(int parts, const std::function<void(int)>& f) {
    std::unique_lock<std::mutex> l(mu_);
    job_ = &f;
    parts_ = parts;
    next_ = 0;
    done_ = 0;
    gen_++;
    cv_.notify_all();
    done_cv_.wait(l, [&] { return done_ == parts_; });
    job_ = nullptr;
  }

 private:
  void run() {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> l(mu_);
    for (;;) {
      cv_.wait(l, [&] { return stop_ || (gen_ != seen && job_ && next_ < parts_); });
      if (stop_) return;
      while (job_ && next_ < parts_) {
        const int i = next_++;
        const std::function<void(int)>* f = job_;
        l.unlock();
        (*f)(i);
        l.lock();
        if (++done_ == parts_) done_cv_.notify_all();
      }
      seen = gen_;
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* job_ = nullptr;
  int parts_ = 0, next_ = 0, done_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

void par_memcpy(Pool& pool, void* dst, const void* src, size_t bytes) {
  const int parts = bytes < (size_t(1) << 20) ? 1 : 2 * pool.size();
  if (parts == 1) {
    memcpy(dst, src, bytes);
    return;
  }
  const size_t step = ((bytes + parts - 1) / parts + 4095) & ~size_t(4095);
  pool.parallel(parts, [&](int i) {
    const size_t a = std::min(bytes, (size_t)i * step), b = std::min(bytes, a + step);
    if (b > a) memcpy((char*)dst + a, (const char*)src + a, b - a);
  });
}

// Process-wide staging state: pinned slots (portable across devices) and
// the worker pool; per device, the matching device slots and a copy stream.
struct DevState {
  void* dslot[NSLOT] = {};
  cudaStream_t copy = nullptr;
  cudaEvent_t ev[NSLOT] = {};
  void* dmap = nullptr;  // column maps of hsrq_pack_download
  size_t dmap_bytes = 0;
};
struct State {
  std::mutex mu;  // one host-I/O call at a time
  void* hslot[NSLOT] = {};
  Pool* pool = nullptr;
  DevState dev[MAX_DEVICES];
};
State& state() {
  static State s;
  return s;
}

bool ensure(State& S, int dev) {
  if (!S.pool) {
    const unsigned hc = std::thread::hardware_concurrency();
    S.pool = new Pool((int)std::max(2u, std::min(16u, hc ? hc : 8u)));
  }
  for (int i = 0; i < NSLOT; i++) {
    if (!S.hslot[i] && !ck(cudaHostAlloc(&S.hslot[i], SLOT_BYTES, cudaHostAllocPortable), "pinned slot"))
      return false;
  }
  DevState& D = S.dev[dev];
  if (!D.copy) {
    if (!ck(cudaStreamCreateWithFlags(&D.copy, cudaStreamNonBlocking), "hostio stream")) return false;
    for (int i = 0; i < NSLOT; i++) {
      if (!ck(cudaMalloc(&D.dslot[i], SLOT_BYTES), "device slot") ||
          !ck(cudaEventCreateWithFlags(&D.ev[i], cudaEventDisableTiming), "hostio event"))
        return false;
    }
  }
  return true;
}

// C-order row block (rows r0.., nr rows, n columns, row-major in `src`) ->
// columns of the column-major H: H[c * ldh + r0 + i] = src[i * n + c].
__global__ void k_rows_to_cols(const double* __restrict__ src, int64_t nr, int64_t n,
                               double* __restrict__ H, int64_t ldh, int64_t r0) {
  __shared__ double t[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32, i0 = (int64_t)blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t i = i0 + k, c = c0 + threadIdx.x;
    if (i < nr && c < n) t[k][threadIdx.x] = src[i * n + c];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t c = c0 + k, i = i0 + threadIdx.x;
    if (i < nr && c < n) H[c * ldh + r0 + i] = t[threadIdx.x][k];
  }
}

// Per row i: s_i = sum_j |h_ij| left to right (numpy's order on an F-order
// array), the subdiagonal entry, and nonzeros at j <= i - 2.  out: [0] =
// max_i s_i as ordered bits (atomicMax; NaN propagates like np.max), [1] =
// structure violations, [2] = zero subdiagonal entries.
__global__ void k_hcheck(const double* __restrict__ H, int64_t ldh, int64_t n,
                         unsigned long long* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  int64_t low = 0;
  const double* p = H + i;
  int64_t j = 0;
  for (; j + 8 <= n; j += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; u++) v[u] = p[(j + u) * ldh];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      s = s + fabs(v[u]);
      if (j + u <= i - 2 && v[u] != 0.0) low++;
    }
  }
  for (; j < n; j++) {
    const double v = p[j * ldh];
    s = s + fabs(v);
    if (j <= i - 2 && v != 0.0) low++;
  }
  unsigned long long key = (unsigned long long)__double_as_longlong(s);
  if (s != s) key = 0x7ff8000000000000ULL;  // canonical NaN: above every number
  atomicMax(&out[0], key);
  if (low) atomicAdd(&out[1], (unsigned long long)low);
  if (i >= 1 && p[(i - 1) * ldh] == 0.0) atomicAdd(&out[2], 1ULL);
}

// Rows [r0, r0 + nr) of the caller's (n, m) output: out[(r - r0) * m + j] =
// (X[re[j] * ldx + r], sgn[j] * X[im[j] * ldx + r]) (complex128, im[j] < 0:
// imaginary part 0) or X[re[j] * ldx + r] (float64).  32 x 32 tiles
// through shared memory so both the X reads (along r) and the output
// writes (along j) are coalesced.
template <bool CPLX>
__global__ void k_pack(const double* __restrict__ X, int64_t ldx, const int64_t* __restrict__ re,
                       const int64_t* __restrict__ im, const double* __restrict__ sgn, int64_t m,
                       int64_t r0, int64_t nr, double* __restrict__ out) {
  __shared__ double tr[32][33];
  __shared__ double ti[CPLX ? 32 : 1][33];
  const int64_t j0 = (int64_t)blockIdx.x * 32, i0 = (int64_t)blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t j = j0 + k, i = i0 + threadIdx.x;
    if (j < m && i < nr) {
      tr[k][threadIdx.x] = X[re[j] * ldx + r0 + i];
      if (CPLX) {
        const int64_t c = im[j];
        ti[k][threadIdx.x] = c >= 0 ? sgn[j] * X[c * ldx + r0 + i] : 0.0;
      }
    }
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t i = i0 + k, j = j0 + threadIdx.x;
    if (j < m && i < nr) {
      if (CPLX) {
        double2 v;
        v.x = tr[threadIdx.x][k];
        v.y = ti[threadIdx.x][k];
        reinterpret_cast<double2*>(out)[i * m + j] = v;
      } else {
        out[i * m + j] = tr[threadIdx.x][k];
      }
    }
  }
}

}  // namespace hostio

extern "C" {

int64_t hsrq_h_upload(const double* h_host, int32_t order, int64_t n, double* H, int64_t ldh,
                      double* checks_host, void* stream_) {
  using namespace hostio;
  if (n < 1 || ldh < n || !h_host || !H || (order != 0 && order != 1)) {
    snprintf(g_err, sizeof(g_err), "hsrq_h_upload: bad arguments");
    return HSRQ_ERR_CONFIG;
  }
  cudaStream_t stream = (cudaStream_t)stream_;
  const int dev = current_device();
  if (dev < 0 || dev >= MAX_DEVICES) return HSRQ_ERR_CONFIG;
  State& S = state();
  std::lock_guard<std::mutex> lock(S.mu);
  if (!ensure(S, dev)) return HSRQ_ERR_CUDA;
  DevState& D = S.dev[dev];
  // the copy stream starts after whatever the caller queued on `stream`
  cudaEvent_t start = D.ev[0];
  if (!ck(cudaEventRecord(start, stream), "record") || !ck(cudaStreamWaitEvent(D.copy, start, 0), "wait"))
    return HSRQ_ERR_CUDA;
  const size_t line = sizeof(double) * (size_t)n;  // one column (F) / row (C) of h
  const int64_t per = std::max<int64_t>(1, (int64_t)(SLOT_BYTES / line));
  int slot = 0;
  bool used[NSLOT] = {};
  for (int64_t a = 0; a < n; a += per) {
    const int64_t b = std::min(n, a + per);
    // the slot's previous copy (and transpose) must be done before reuse
    if (used[slot] && !ck(cudaEventSynchronize(D.ev[slot]), "slot wait")) return HSRQ_ERR_CUDA;
    par_memcpy(*S.pool, S.hslot[slot], (const char*)h_host + (size_t)a * line, (size_t)(b - a) * line);
    if (order == 1) {  // F-order: columns a..b-1 straight into H (ld padding)
      if (!ck(cudaMemcpy2DAsync(H + a * ldh, sizeof(double) * ldh, S.hslot[slot], line, line,
                                (size_t)(b - a), cudaMemcpyHostToDevice, D.copy),
              "H2D H"))
        return HSRQ_ERR_CUDA;
    } else {  // C-order: rows a..b-1 = columns of H^T; transpose on the device
      if (!ck(cudaMemcpyAsync(D.dslot[slot], S.hslot[slot], (size_t)(b - a) * line,
                              cudaMemcpyHostToDevice, D.copy),
              "H2D H rows"))
        return HSRQ_ERR_CUDA;
      const dim3 grid((unsigned)((n + 31) / 32), (unsigned)((b - a + 31) / 32));
      k_rows_to_cols<<<grid, dim3(32, 8), 0, D.copy>>>((const double*)D.dslot[slot], b - a, n, H,
                                                        ldh, a);
    }
    if (!ck(cudaEventRecord(D.ev[slot], D.copy), "record slot")) return HSRQ_ERR_CUDA;
    used[slot] = true;
    slot = (slot + 1) % NSLOT;
  }
  // checks on the compute stream, after the copies
  unsigned long long* chk = (unsigned long long*)D.dslot[slot];
  if (used[slot] && !ck(cudaEventSynchronize(D.ev[slot]), "slot wait")) return HSRQ_ERR_CUDA;
  if (!ck(cudaMemsetAsync(chk, 0, 3 * sizeof(unsigned long long), D.copy), "memset")) return HSRQ_ERR_CUDA;
  k_hcheck<<<(unsigned)((n + 127) / 128), 128, 0, D.copy>>>(H, ldh, n, chk);
  unsigned long long r[3];
  if (!ck(cudaMemcpyAsync(r, chk, sizeof(r), cudaMemcpyDeviceToHost, D.copy), "D2H checks") ||
      !ck(cudaEventRecord(D.ev[slot], D.copy), "record") ||
      !ck(cudaStreamWaitEvent(stream, D.ev[slot], 0), "join") ||
      !ck(cudaStreamSynchronize(D.copy), "sync"))
    return HSRQ_ERR_CUDA;
  memcpy(&checks_host[0], &r[0], sizeof(double));
  checks_host[1] = (double)r[1];
  checks_host[2] = (double)r[2];
  return 0;
}

int64_t hsrq_host_prefault(void* ptr, int64_t bytes, int32_t threads) {
  // Touch one byte per 4 KiB page of a fresh (untouched) host allocation
  // from `threads` threads, so the page faults are taken while the GPU works
  // rather than inside hsrq_pack_download's copies.  Own threads (not the
  // pool): callers run this concurrently with the upload / solve.
  if (!ptr || bytes < 0 || threads < 1) return HSRQ_ERR_CONFIG;
  const size_t page = 4096, total = (size_t)bytes;
  const size_t per = ((total / threads + page - 1) / page) * page;
  std::vector<std::thread> th;
  for (int t = 0; t < threads; t++) {
    const size_t a = std::min(total, (size_t)t * per), b = std::min(total, a + per);
    if (b <= a) break;
    th.emplace_back([=] {
      volatile char* p = (volatile char*)ptr;
      for (size_t o = a; o < b; o += page) p[o] = 0;
    });
  }
  for (auto& t : th) t.join();
  return 0;
}

int64_t hsrq_pack_download(const double* X, int64_t ldx, int64_t n, int64_t m,
                           const int64_t* re_col, const int64_t* im_col, const double* im_sign,
                           int32_t cplx_out, void* out_host, void* stream_) {
  using namespace hostio;
  if (n < 1 || m < 1 || ldx < n || !X || !re_col || !out_host || (cplx_out && (!im_col || !im_sign))) {
    snprintf(g_err, sizeof(g_err), "hsrq_pack_download: bad arguments");
    return HSRQ_ERR_CONFIG;
  }
  cudaStream_t stream = (cudaStream_t)stream_;
  const int dev = current_device();
  if (dev < 0 || dev >= MAX_DEVICES) return HSRQ_ERR_CONFIG;
  State& S = state();
  std::lock_guard<std::mutex> lock(S.mu);
  if (!ensure(S, dev)) return HSRQ_ERR_CUDA;
  DevState& D = S.dev[dev];
  const size_t mapb = sizeof(int64_t) * 2 * m + sizeof(double) * m;
  if (D.dmap_bytes < mapb) {
    if (D.dmap) cudaFree(D.dmap);
    D.dmap = nullptr;
    D.dmap_bytes = 0;
    if (!ck(cudaMalloc(&D.dmap, mapb), "map alloc")) return HSRQ_ERR_CUDA;
    D.dmap_bytes = mapb;
  }
  int64_t* dre = (int64_t*)D.dmap;
  int64_t* dim = dre + m;
  double* dsg = (double*)(dim + m);
  if (!ck(cudaMemcpyAsync(dre, re_col, sizeof(int64_t) * m, cudaMemcpyHostToDevice, stream), "H2D map") ||
      (cplx_out &&
       (!ck(cudaMemcpyAsync(dim, im_col, sizeof(int64_t) * m, cudaMemcpyHostToDevice, stream), "H2D map") ||
        !ck(cudaMemcpyAsync(dsg, im_sign, sizeof(double) * m, cudaMemcpyHostToDevice, stream), "H2D map"))))
    return HSRQ_ERR_CUDA;
  const size_t row = (cplx_out ? 16 : 8) * (size_t)m;  // bytes of one output row
  const int64_t per = std::max<int64_t>(1, (int64_t)(SLOT_BYTES / row));
  if ((size_t)per * row > SLOT_BYTES) {
    snprintf(g_err, sizeof(g_err), "hsrq_pack_download: m too large for a staging slot");
    return HSRQ_ERR_CONFIG;
  }
  // pack on `stream` (after the solve), D2H on the copy stream; the host
  // copies out of slot s run while the device packs / copies the next ones
  struct Pending {
    int64_t a, b;
    int slot;
  };
  std::vector<Pending> q;
  int slot = 0;
  bool used[NSLOT] = {};
  auto drain = [&](const Pending& p) -> bool {
    if (!ck(cudaEventSynchronize(D.ev[p.slot]), "d2h wait")) return false;
    par_memcpy(*S.pool, (char*)out_host + (size_t)p.a * row, S.hslot[p.slot], (size_t)(p.b - p.a) * row);
    return true;
  };
  for (int64_t a = 0; a < n; a += per) {
    const int64_t b = std::min(n, a + per);
    if (used[slot]) {  // slot busy: finish its host copy first
      if (!drain(q.front())) return HSRQ_ERR_CUDA;
      q.erase(q.begin());
    }
    const dim3 grid((unsigned)((m + 31) / 32), (unsigned)((b - a + 31) / 32));
    if (cplx_out)
      k_pack<true><<<grid, dim3(32, 8), 0, stream>>>(X, ldx, dre, dim, dsg, m, a, b - a,
                                                     (double*)D.dslot[slot]);
    else
      k_pack<false><<<grid, dim3(32, 8), 0, stream>>>(X, ldx, dre, dim, dsg, m, a, b - a,
                                                      (double*)D.dslot[slot]);
    if (!ck(cudaGetLastError(), "k_pack") || !ck(cudaEventRecord(D.ev[slot], stream), "record") ||
        !ck(cudaStreamWaitEvent(D.copy, D.ev[slot], 0), "wait") ||
        !ck(cudaMemcpyAsync(S.hslot[slot], D.dslot[slot], (size_t)(b - a) * row,
                            cudaMemcpyDeviceToHost, D.copy),
            "D2H pack") ||
        !ck(cudaEventRecord(D.ev[slot], D.copy), "record"))
      return HSRQ_ERR_CUDA;
    q.push_back({a, b, slot});
    used[slot] = true;
    slot = (slot + 1) % NSLOT;
  }
  for (const Pending& p : q)
    if (!drain(p)) return HSRQ_ERR_CUDA;
  // later work on `stream` may overwrite X only after the last pack read it
  return 0;
}

}  // extern "C"
