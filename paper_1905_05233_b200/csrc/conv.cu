// conv.cu -- C-ABI device entry points of the 2D layer (include/wino.h):
// wino_conv2d = K2 weight transform -> K1 input transform -> K3 tcgen05
// Winograd-domain GEMM -> K4 output transform, all on the caller's stream.
#include <cstdlib>
#include <string>

#include "device.cuh"
#include "geometry.hpp"

namespace wino {
wino_status run_weight_transform(const void* w, int K, int C, const wino_algo* al, wino_dtype dt, void* U,
                                 cudaStream_t st);
wino_status run_input_transform(const void* x, int N, int C, int H, int W, int pad, const wino_algo* al,
                                wino_dtype dt, wino_layout layout, void* V, cudaStream_t st);
wino_status run_domain_gemm(const void* V, const void* U, const Geo& g, const wino_algo* al, wino_dtype dt,
                            void* M, cudaStream_t st, int mb0 = 0, int nT = -1);
wino_status run_domain_gemm_split(const void* V, const void* U, const Geo& g, const wino_algo* al, wino_dtype dt,
                                  float* M, void* y, int* cnt, cudaStream_t st);
wino_status run_output_transform(const void* Mw, int N, int K, int H, int W, int pad, const wino_algo* al,
                                 wino_dtype dt, wino_layout layout, void* y, cudaStream_t st, int t0 = 0,
                                 int nT = -1, int Tpm = 0, int disc = 0);
}  // namespace wino

using namespace wino;

// The fused K3+K4 kernel (output transform from L2, gemm.cu) is opt-in with
// WINO_FUSED=1: on B200 its fixup warps are L2-latency bound and the staged
// K3 -> K4 pair is faster, so the staged pair is the default.
static bool fused_disabled() {
  static const int v = [] {
    const char* e = getenv("WINO_FUSED");
    return e && *e && *e != '0' ? 0 : 1;
  }();
  return v != 0;
}

static wino_status check_layer(const wino_algo* al, int N, int C, int H, int W, int K, int pad, wino_dtype dt,
                               wino_layout layout) {
  if (!al) return set_last_error("NULL algo"), WINO_E_ARG;
  if (N <= 0 || C <= 0 || K <= 0 || (pad != 0 && pad != 1) || H + 2 * pad < 3 || W + 2 * pad < 3)
    return set_last_error("bad layer geometry (need N, C, K > 0, pad in {0,1}, H, W + 2 pad >= 3)"), WINO_E_ARG;
  if (dt != WINO_F32 && dt != WINO_F16 && dt != WINO_BF16) return set_last_error("bad dtype"), WINO_E_ARG;
  if (layout != WINO_NCHW && layout != WINO_NHWC) return set_last_error("bad layout"), WINO_E_ARG;
  if (al->r != 3) return set_last_error("r != 3"), WINO_E_UNSUPPORTED;
  if (K > 65535) return set_last_error("K > 65535 unsupported"), WINO_E_UNSUPPORTED;
  return WINO_OK;
}

extern "C" {

wino_status wino_conv2d_workspace(const wino_algo* al, int N, int C, int H, int W, int K, int pad,
                                  wino_dtype dt, wino_layout layout, size_t* bytes) {
  if (!bytes) return set_last_error("NULL bytes"), WINO_E_ARG;
  wino_status s = check_layer(al, N, C, H, W, K, pad, dt, layout);
  if (s != WINO_OK) return s;
  *bytes = make_geo(al, N, C, H, W, K, pad, dt).total;
  return WINO_OK;
}

// Tile blocks per K3 -> K4 slice (0: one pass over the whole layer).  Opt-in
// (WINO_CHUNK_TB=<blocks>, or "auto": slices of M of about 40 MB, well inside the
// 126 MB L2); NCHW output only.
static int chunk_blocks(const Geo& g, wino_layout layout) {
  static const char* e = getenv("WINO_CHUNK_TB");
  if (!e || layout != WINO_NCHW) return 0;
  if (std::string(e) == "auto") {
    const size_t blk = (size_t)g.Q * g.K * 128 * 4;   // M bytes per tile block
    const int cb = (int)((40u << 20) / (blk ? blk : 1));
    return cb < 1 ? 1 : cb;
  }
  return atoi(e);
}

wino_status wino_conv2d(const void* x, const void* w, int N, int C, int H, int W, int K, int pad,
                        const wino_algo* al, wino_dtype dt, wino_layout layout, void* out, void* ws,
                        size_t ws_bytes, void* stream) {
  reset_launch_count();
  wino_status s = check_layer(al, N, C, H, W, K, pad, dt, layout);
  if (s != WINO_OK) return s;
  if (!x || !w || !out || !ws) return set_last_error("NULL buffer"), WINO_E_ARG;
  if (reinterpret_cast<uintptr_t>(ws) % 1024) return set_last_error("workspace must be 1024-byte aligned"), WINO_E_ARG;
  Geo g = make_geo(al, N, C, H, W, K, pad, dt);
  if (ws_bytes < g.total) return set_last_error("workspace too small"), WINO_E_WORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  char* base = static_cast<char*>(ws);
  void* U = base + g.offU;
  void* V = base + g.offV;
  float* M = reinterpret_cast<float*>(base + g.offM);
  // K2 (weights) and K1 (inputs) are independent: K2 runs on a library-owned
  // side stream forked from and joined back into the caller's stream (events,
  // so the pair stays CUDA-graph capturable), overlapping K1's start.
  DevState* ds = dev_state();   // per (thread, device): the caller's stream must be on the current device
  if (!ds) return WINO_E_CUDA;
  cudaEvent_t ev_fork = ds->fork, ev_join = ds->join;
  cudaStream_t s_w = ds->side;
  WINO_CUDA_CHECK(cudaEventRecord(ev_fork, st));
  WINO_CUDA_CHECK(cudaStreamWaitEvent(s_w, ev_fork, 0));
  if ((s = run_weight_transform(w, K, C, al, dt, U, s_w)) != WINO_OK) return s;
  WINO_CUDA_CHECK(cudaEventRecord(ev_join, s_w));
  if ((s = run_input_transform(x, N, C, H, W, pad, al, dt, layout, V, st)) != WINO_OK) return s;
  WINO_CUDA_CHECK(cudaStreamWaitEvent(st, ev_join, 0));
  const bool m16 = m_in_dtype(al, dt);   // M3: the opt-in fused / chunked paths keep an fp32 M
  if (layout == WINO_NCHW && !fused_disabled() && !m16) {
    s = run_domain_gemm_split(V, U, g, al, dt, M, out, reinterpret_cast<int*>(base + g.offD), st);
    if (s != WINO_E_UNSUPPORTED) return s;   // OK or a real failure
  }
  const int cb = m16 ? 0 : chunk_blocks(g, layout);
  if (cb > 0 && cb < g.TB) {
    // K3 -> K4 per slice of cb tile blocks through one L2-sized M slice that K4
    // discards after reading: M never travels to HBM (see chunk_blocks)
    for (int mb0 = 0; mb0 < g.TB; mb0 += cb) {
      const int nT = (g.T - mb0 * 128) < cb * 128 ? g.T - mb0 * 128 : cb * 128;
      if ((s = run_domain_gemm(V, U, g, al, dt, M, st, mb0, nT)) != WINO_OK) return s;
      if ((s = run_output_transform(M, N, K, H, W, pad, al, dt, layout, out, st, mb0 * 128, nT, (nT + 31) / 32 * 32,
                                    1)) != WINO_OK)
        return s;
    }
    return WINO_OK;
  }
  if ((s = run_domain_gemm(V, U, g, al, dt, M, st)) != WINO_OK) return s;
  if ((s = run_output_transform(M, N, K, H, W, pad, al, dt, layout, out, st)) != WINO_OK) return s;
  return WINO_OK;
}

wino_status wino_conv2d_host_io(const void* x_host, void* x_dev, const void* w_dev, int N, int C, int H, int W,
                                int K, int pad, const wino_algo* al, wino_dtype dt, wino_layout layout,
                                void* out_dev, void* out_host, void* ws, size_t ws_bytes, void* stream) {
  wino_status s = check_layer(al, N, C, H, W, K, pad, dt, layout);
  if (s != WINO_OK) return s;
  if (!x_host || !out_host || !x_dev || !out_dev) return set_last_error("NULL buffer"), WINO_E_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Geo g = make_geo(al, N, C, H, W, K, pad, dt);
  if (ws_bytes < g.total) return set_last_error("workspace too small"), WINO_E_WORKSPACE;
  // Images are independent (P:498 tiles never cross images), so the batch is
  // processed in chunks: the H2D copy of chunk j+1 and the D2H copy of chunk j-1
  // (two library-owned copy streams, opposite PCIe directions) overlap the layer
  // on chunk j (the caller's stream).  The layer is far faster than PCIe, so
  // the time is the copies plus the pipeline's fill and drain -- the first
  // chunk's H2D and the last chunk's D2H.  Chunk sizes therefore ramp up
  // geometrically from one image to N/8 and back down (1, 1, 2, 2, 4, 4, ...
  // ..., 4, 2, 1), which makes the fill and drain a few images long.  The
  // caller's stream finally waits for the last copy, so synchronising it
  // covers everything.
  const size_t xi = (size_t)C * H * W * g.es, yi = (size_t)K * g.Ho * g.Wo * g.es;   // bytes per image
  int plan[63], nch = 0;
  {
    static const int kUniform = [] {   // tuning knob: WINO_HOSTIO_CHUNKS=<n> equal chunks instead
      const char* e = getenv("WINO_HOSTIO_CHUNKS");
      const int v = e ? atoi(e) : 0;
      return v < 0 ? 0 : (v > 63 ? 63 : v);
    }();
    if (kUniform) {
      nch = N >= kUniform ? kUniform : N;
      for (int j = 0; j < nch; ++j) plan[j] = N / nch + (j < N % nch ? 1 : 0);
    } else {
      int head[32], tail[32], nh = 0, nt = 0, rem = N, sz = 1;
      const int cap = N / 8 > 1 ? N / 8 : 1;
      while (rem > 0 && nh + nt < 61) {
        head[nh] = sz < rem ? sz : rem, rem -= head[nh++];
        if (rem <= 0) break;
        tail[nt] = sz < rem ? sz : rem, rem -= tail[nt++];
        if (sz < cap) sz = 2 * sz < cap ? 2 * sz : cap;
      }
      for (int j = 0; j < nh; ++j) plan[nch++] = head[j];
      if (rem > 0) plan[nch++] = rem;   // (chunk-count limit reached)
      for (int j = nt - 1; j >= 0; --j) plan[nch++] = tail[j];
    }
  }
  DevState* ds = dev_state();
  if (!ds) return WINO_E_CUDA;
  cudaStream_t s_in = ds->io_in, s_out = ds->io_out;
  cudaEvent_t(&ev)[2][64] = ds->io_ev;
  // copies must not start before work already queued on the caller's stream
  cudaEvent_t start = ev[1][63];
  WINO_CUDA_CHECK(cudaEventRecord(start, st));
  WINO_CUDA_CHECK(cudaStreamWaitEvent(s_in, start, 0));
  WINO_CUDA_CHECK(cudaStreamWaitEvent(s_out, start, 0));
  int launches = 0;
  for (int j = 0, n0 = 0; j < nch; ++j) {
    const int nj = plan[j];
    char* xd = static_cast<char*>(x_dev) + (size_t)n0 * xi;
    char* yd = static_cast<char*>(out_dev) + (size_t)n0 * yi;
    WINO_CUDA_CHECK(cudaMemcpyAsync(xd, static_cast<const char*>(x_host) + (size_t)n0 * xi, (size_t)nj * xi,
                                    cudaMemcpyHostToDevice, s_in));
    WINO_CUDA_CHECK(cudaEventRecord(ev[0][j], s_in));
    WINO_CUDA_CHECK(cudaStreamWaitEvent(st, ev[0][j], 0));
    s = wino_conv2d(xd, w_dev, nj, C, H, W, K, pad, al, dt, layout, yd, ws, ws_bytes, stream);
    if (s != WINO_OK) return s;
    launches += wino_last_launch_count();
    WINO_CUDA_CHECK(cudaEventRecord(ev[1][j], st));
    WINO_CUDA_CHECK(cudaStreamWaitEvent(s_out, ev[1][j], 0));
    WINO_CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(out_host) + (size_t)n0 * yi, yd, (size_t)nj * yi,
                                    cudaMemcpyDeviceToHost, s_out));
    n0 += nj;
  }
  WINO_CUDA_CHECK(cudaEventRecord(ev[0][63], s_out));
  WINO_CUDA_CHECK(cudaStreamWaitEvent(st, ev[0][63], 0));
  reset_launch_count();
  count_launch(launches);
  return WINO_OK;
}

wino_status wino_weight_transform(const void* w, int K, int C, const wino_algo* al, wino_dtype dt, void* U,
                                  void* stream) {
  reset_launch_count();
  wino_status s = check_layer(al, 1, C, 3, 3, K, 0, dt, WINO_NCHW);
  if (s != WINO_OK) return s;
  if (!w || !U) return set_last_error("NULL buffer"), WINO_E_ARG;
  return run_weight_transform(w, K, C, al, dt, U, reinterpret_cast<cudaStream_t>(stream));
}

wino_status wino_input_transform(const void* x, int N, int C, int H, int W, int pad, const wino_algo* al,
                                 wino_dtype dt, wino_layout layout, void* V, void* stream) {
  reset_launch_count();
  wino_status s = check_layer(al, N, C, H, W, 1, pad, dt, layout);
  if (s != WINO_OK) return s;
  if (!x || !V) return set_last_error("NULL buffer"), WINO_E_ARG;
  return run_input_transform(x, N, C, H, W, pad, al, dt, layout, V, reinterpret_cast<cudaStream_t>(stream));
}

wino_status wino_domain_gemm(const void* V, const void* U, int T, int C, int K, const wino_algo* al,
                             wino_dtype dt, void* M, void* stream) {
  reset_launch_count();
  if (!al || !V || !U || !M || T <= 0 || C <= 0 || K <= 0) return set_last_error("bad argument"), WINO_E_ARG;
  if (reinterpret_cast<uintptr_t>(V) % 16 || reinterpret_cast<uintptr_t>(U) % 16)
    return set_last_error("V and U must be 16-byte aligned"), WINO_E_ARG;
  Geo g = make_geo(al, 1, C, 3, 3, K, 0, dt);  // Cp, Q, S, es, planes
  g.T = T;
  g.Tp = (int)align_up(T, 32);
  g.TB = (T + 127) / 128;
  return run_domain_gemm(V, U, g, al, dt, M, reinterpret_cast<cudaStream_t>(stream));
}

wino_status wino_output_transform(const void* M, int N, int K, int H, int W, int pad, const wino_algo* al,
                                  wino_dtype dt, wino_layout layout, void* out, void* stream) {
  reset_launch_count();
  wino_status s = check_layer(al, N, 1, H, W, K, pad, dt, layout);
  if (s != WINO_OK) return s;
  if (!M || !out) return set_last_error("NULL buffer"), WINO_E_ARG;
  return run_output_transform(M, N, K, H, W, pad, al, dt, layout, out, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
