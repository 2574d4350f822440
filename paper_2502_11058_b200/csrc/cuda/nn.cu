// nn.cu — the NN local step of DreamDDP on sm_100a (include/dsx_nn.h):
// a K-worker MLP (Linear + ReLU stack, softmax cross-entropy) whose local
// step is FP -> loss -> BP with the optimizer fused per layer, and whose
// scheduled layers are averaged across all K workers on a side stream as
// soon as BP(l) + update(l) finished (Alg. 1), so the
// average overlaps BP(l-1..1).
//
// Layout (one rank, kl local workers):
//   params   fp32 [kl][P]   layer l: W_l[out][in] at off_l (64-element
//                           aligned), b_l[out] right after; a sync set is
//                           one contiguous range per worker
//   pbf      bf16 [kl][P]   the GEMM copy of params (bf16 mode)
//   grads    fp32 [kl][P]   dW (wgrad epilogue), db (column sums)
//   mom, var fp32 [kl][P]   optimizer states (local, never averaged)
//   act[l]   T [kl][batch][width_l]   layer inputs (act[0] = x); logits fp32
//   dz[2]    T [kl][batch][max width] gradient ping-pong
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "dsx.h"
#include "dsx_nn.h"
#include "nn_gemm.cuh"
#include "nn_kernels.cuh"

namespace dsx {
extern thread_local std::string g_last_error;
}

namespace dsx_nn {
namespace {

dsx_status nfail(dsx_status code, const std::string& msg) {
  dsx::g_last_error = msg;
  return code;
}

#define NN_CUDA(expr)                                                                           \
  do {                                                                                          \
    cudaError_t e_ = (expr);                                                                    \
    if (e_ != cudaSuccess) return nfail(DSX_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)
#define NN_NCCL(expr)                                                                           \
  do {                                                                                          \
    ncclResult_t r_ = (expr);                                                                   \
    if (r_ != ncclSuccess) return nfail(DSX_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(r_)); \
  } while (0)
#define NN_TRY(expr)              \
  do {                            \
    dsx_status s_ = (expr);       \
    if (s_ != DSX_OK) return s_;  \
  } while (0)

}  // namespace


}  // namespace dsx_nn

using namespace dsx_nn;

struct dsx_mlp {
  int device = 0;
  bool bf16 = false;
  int K = 1, kbegin = 0, kl = 1;
  int L = 0;
  std::vector<int> widths;
  int batch = 0;
  int opt = DSX_OPT_SGD;
  float mu = 0.9f, b1 = 0.9f, b2 = 0.999f, eps = 1e-8f, wd = 0.f;
  int nsm = 148;

  std::vector<long long> off;      // device layout: layer l W at off[l-1], b at boff[l-1]
  std::vector<long long> boff;
  std::vector<long long> packed;   // host packed layout offsets [L+1]
  long long P = 0;                 // device arena stride per worker (elements)
  float* params = nullptr;
  __nv_bfloat16* pbf = nullptr;
  float* grads = nullptr;
  float* mom = nullptr;
  float* var = nullptr;
  std::vector<void*> act;          // [L]: inputs of layer l+1 (T), act[0] = x
  float* logits = nullptr;         // [kl][batch][C]
  void* dz[2] = {nullptr, nullptr};
  int maxw = 0;
  float* xin = nullptr;            // fp32 staging of host x [kl][batch][in]
  int* labels = nullptr;
  const int* labels_dev = nullptr; // labels the next step reads
  const float* x_dev = nullptr;    // device x the next step reads (fp32)
  float* loss_part = nullptr;
  float* loss = nullptr;

  cudaStream_t stream = nullptr, side = nullptr;
  std::vector<cudaEvent_t> ev_upd, ev_sync;
  std::vector<unsigned char> synced_prev;  // layer l averaged last step (FP(l) must wait)
  cudaEvent_t ev[8] = {};
  cudaEvent_t iev[4] = {};   // step start, compute done, sync done (side), step end
  bool instrument = false;
  bool any_synced = false;
  uint64_t launches = 0;

  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  double link_bw = 0.0, link_lat = 0.0;  // throttled link (bw <= 0: off)
  bool overlap = true;                   // false: averages after the whole BP (ssgd/flsgd modes)
  // per-step scalars: device copy + pinned ring of host slots (one per step
  // in flight); CUDA graphs, one per distinct sync mask
  dsx_nn::StepDev* sp = nullptr;
  dsx_nn::StepDev* ring = nullptr;
  std::vector<cudaEvent_t> ring_ev;
  unsigned long long ring_i = 0;
  bool graphs = false;
  bool side_used = false;                // the last step_impl put work on the sync stream
  struct Graph {
    cudaGraphExec_t exec = nullptr;
    uint64_t launches = 0;
  };
  std::vector<std::pair<std::string, Graph>> graph_cache;
  // events used only inside captures (an event recorded in a capture cannot
  // be waited on eagerly afterwards), and the pre-capture drain
  std::vector<cudaEvent_t> gev_upd, gev_sync;
  cudaEvent_t ev_join = nullptr, ev_drain = nullptr;
  // several ranks: the step graph holds only the compute; it records hev_upd[l]
  // as external event nodes and the NCCL averages are issued eagerly on the
  // side stream behind them (capturing the collectives hung at 2 GPUs)
  std::vector<cudaEvent_t> hev_upd;
};

namespace dsx_nn {
namespace {

size_t esz(const dsx_mlp* m) { return m->bf16 ? 2 : 4; }
// row pitch of a gradient of width widths[i]: 16-B rows for TMA in bf16 mode
// (only the class count may be unaligned; padding columns are never read:
// the tensor maps use the logical width)
long long ldz(const dsx_mlp* m, int i) {
  const long long w = m->widths[i];
  return m->bf16 ? (w + 7) / 8 * 8 : w;
}

dsx_status check(dsx_mlp* m) {
  if (!m) return nfail(DSX_ERR_ARGUMENT, "null mlp");
  NN_CUDA(cudaSetDevice(m->device));
  return DSX_OK;
}


// average of layer l's range over all K workers, on stream s
dsx_status average_layer(dsx_mlp* m, int l, cudaStream_t s) {
  const long long lo = m->off[l], n = m->boff[l] + m->widths[l + 1] - m->off[l];
  std::string err;
  const dsx_status st = average_range(m->params, m->bf16 ? m->pbf : nullptr, m->P, m->kl, m->K, m->nranks, m->comm,
                                      lo, n, m->nsm, s, &m->launches, &err);
  if (st != DSX_OK) return nfail(st, err);
  NN_CUDA(cudaGetLastError());
  return DSX_OK;
}

GemmCall base_call(const dsx_mlp* m) {
  GemmCall c{};
  c.bf16 = m->bf16;
  c.out_bf16 = m->bf16;
  c.g.batch = m->kl;
  return c;
}

// FP of layer l (0-based): act[l] -> act[l+1] (or logits)
dsx_status forward_layer(dsx_mlp* m, int l) {
  const int in = m->widths[l], out = m->widths[l + 1];
  const bool last = l == m->L - 1;
  GemmCall c = base_call(m);
  c.A = m->act[l];
  c.lda = in;
  c.sA = (long long)m->batch * in;
  c.B = m->bf16 ? static_cast<const void*>(m->pbf + m->off[l]) : static_cast<const void*>(m->params + m->off[l]);
  c.ldb = in;
  c.sB = m->P;
  c.g.M = m->batch;
  c.g.N = out;
  c.g.K = in;
  c.g.epi = kEpiBiasAct;
  c.g.relu = last ? 0 : 1;
  c.g.bias = m->params + m->boff[l];
  c.g.strideBias = m->P;
  if (last) {
    c.out_bf16 = false;
    c.g.C = m->logits;
  } else {
    c.g.C = m->act[l + 1];
  }
  c.g.ldc = out;
  c.g.strideC = (long long)m->batch * out;
  ++m->launches;
  return gemm(c, m->stream, m->nsm);
}

// BP of layer l (0-based): dz_cur = dL/d(pre-activation of layer l) ->
// dW, db, (dz_prev), then the optimizer update
dsx_status backward_layer(dsx_mlp* m, int l, void* dz_cur, void* dz_prev, const OptArgs& o, const StepDev* sp) {
  const int in = m->widths[l], out = m->widths[l + 1];
  const long long ld_cur = ldz(m, l + 1), ld_prev = ldz(m, l);
  // wgrad: dW[out][in] = dz^T x : A = dz (M-major), B = x (N-major)
  {
    GemmCall c = base_call(m);
    c.a_mn = true;
    c.b_mn = true;
    c.A = dz_cur;
    c.lda = ld_cur;
    c.sA = (long long)m->batch * m->maxw;
    c.B = m->act[l];
    c.ldb = in;
    c.sB = (long long)m->batch * in;
    c.g.M = out;
    c.g.N = in;
    c.g.K = m->batch;
    c.g.epi = kEpiF32;
    c.g.C = m->grads + m->off[l];
    c.g.ldc = in;
    c.g.strideC = m->P;
    ++m->launches;
    NN_TRY(gemm(c, m->stream, m->nsm));
  }
  // db = column sums of dz
  {
    dim3 grid((out + 31) / 32, m->kl);
    if (m->bf16)
      NN_CUDA(launch_pdl(colsum_kernel<__nv_bfloat16>, grid, 256, 0, m->stream, static_cast<const __nv_bfloat16*>(dz_cur), ld_cur,
                                                                (long long)m->batch * m->maxw, m->batch, out,
                                                                m->grads + m->boff[l], m->P));
    else
      NN_CUDA(launch_pdl(colsum_kernel<float>, grid, 256, 0, m->stream, static_cast<const float*>(dz_cur), ld_cur,
                                                        (long long)m->batch * m->maxw, m->batch, out,
                                                        m->grads + m->boff[l], m->P));
    ++m->launches;
  }
  // dgrad through the ReLU of layer l-1's output: dz_prev = (dz W) * (x > 0)
  if (l > 0) {
    GemmCall c = base_call(m);
    c.a_mn = false;
    c.b_mn = true;
    c.A = dz_cur;
    c.lda = ld_cur;
    c.sA = (long long)m->batch * m->maxw;
    c.B = m->bf16 ? static_cast<const void*>(m->pbf + m->off[l]) : static_cast<const void*>(m->params + m->off[l]);
    c.ldb = in;
    c.sB = m->P;
    c.g.M = m->batch;
    c.g.N = in;
    c.g.K = out;
    c.g.epi = kEpiDRelu;
    c.g.mask = m->act[l];
    c.g.ldmask = in;
    c.g.strideMask = (long long)m->batch * in;
    c.g.C = dz_prev;
    c.g.ldc = ld_prev;
    c.g.strideC = (long long)m->batch * m->maxw;
    ++m->launches;
    NN_TRY(gemm(c, m->stream, m->nsm));
  }
  // the layer's optimizer step (W and b are one contiguous range)
  const long long lo = m->off[l], n = m->boff[l] + out - m->off[l];
  // ~4 resident blocks per SM over all workers, each thread 2 x 16 B per pass
  const long long want = (n / 8 + 255) / 256;
  dim3 grid((unsigned)std::max<long long>(1, std::min<long long>(want, (long long)m->nsm * 8 / m->kl)), m->kl);
  NN_CUDA(launch_pdl(optimizer_kernel, grid, 256, 0, m->stream, m->params, m->grads, m->mom, m->var, m->bf16 ? m->pbf : nullptr, m->P,
                                                lo, n, o, sp));
  ++m->launches;
  NN_CUDA(cudaGetLastError());
  return DSX_OK;
}

// The step's scalars (lr, Adam bias corrections) and batch pointers into the
// device StepDev, through a pinned ring slot (copied on the compute stream, so
// a captured graph replayed after it reads this step's values).
dsx_status write_step(dsx_mlp* m, double lr, long long t) {
  if (!m->x_dev || !m->labels_dev) return nfail(DSX_ERR_STATE, "dsx_mlp_step: no batch set (dsx_mlp_set_batch)");
  const int slot = (int)(m->ring_i++ % m->ring_ev.size());
  NN_CUDA(cudaEventSynchronize(m->ring_ev[slot]));  // the slot's previous copy has run
  StepDev& h = m->ring[slot];
  h.lr = (float)lr;
  h.bc1 = (float)(1.0 - std::pow((double)m->b1, (double)(t + 1)));
  h.bc2 = (float)(1.0 - std::pow((double)m->b2, (double)(t + 1)));
  h.pad = 0.f;
  h.x = m->x_dev;
  h.labels = m->labels_dev;
  NN_CUDA(cudaMemcpyAsync(m->sp, &h, sizeof(StepDev), cudaMemcpyHostToDevice, m->stream));
  NN_CUDA(cudaEventRecord(m->ring_ev[slot], m->stream));
  return DSX_OK;
}

dsx_status prepare_input(dsx_mlp* m) {
  const long long n = (long long)m->kl * m->batch * m->widths[0];
  if (m->bf16)
    NN_CUDA(launch_pdl(load_x_kernel<__nv_bfloat16>, blocks_for(n, m->nsm), 256, 0, m->stream, 
        m->sp, static_cast<__nv_bfloat16*>(m->act[0]), n));
  else
    NN_CUDA(launch_pdl(load_x_kernel<float>, blocks_for(n, m->nsm), 256, 0, m->stream, m->sp, static_cast<float*>(m->act[0]), n));
  ++m->launches;
  return DSX_OK;
}

// one layer's average on the side stream (+ the throttled link's busy time)
dsx_status side_sync(dsx_mlp* m, int l) {
  NN_TRY(average_layer(m, l, m->side));
  if (m->link_bw > 0.0) {
    const double bytes = 4.0 * (double)(m->boff[l] + m->widths[l + 1] - m->off[l]);
    nn_link_spin_kernel<<<1, 1, 0, m->side>>>((unsigned long long)((m->link_lat + bytes / m->link_bw) * 1e9));
    ++m->launches;
  }
  return DSX_OK;
}

// capturing && hybrid: the compute only, with external event records where
// the averages start (issued eagerly after the launch: issue_hybrid_syncs)
dsx_status step_impl(dsx_mlp* m, double lr, long long t, const unsigned char* mask, bool capturing,
                     bool hybrid = false) {
  OptArgs o{};
  o.kind = m->opt;
  o.lr = (float)lr;
  o.mu = m->mu;
  o.b1 = m->b1;
  o.b2 = m->b2;
  o.eps = m->eps;
  o.wd = m->wd;
  o.bc1 = (float)(1.0 - std::pow((double)m->b1, (double)(t + 1)));
  o.bc2 = (float)(1.0 - std::pow((double)m->b2, (double)(t + 1)));
  if (m->instrument) NN_CUDA(cudaEventRecord(m->iev[0], m->stream));
  NN_TRY(prepare_input(m));
  // FP: layer l waits for last step's average of layer l (in place); a
  // replayed graph already joined its averages before it ended
  for (int l = 0; l < m->L; ++l) {
    if (m->synced_prev[l] && !capturing) NN_CUDA(cudaStreamWaitEvent(m->stream, m->ev_sync[l], 0));
    NN_TRY(forward_layer(m, l));
  }
  // loss + dlogits
  {
    const int C = m->widths[m->L];
    dim3 grid((m->batch * 32 + 255) / 256, m->kl);
    if (m->bf16)
      NN_CUDA(launch_pdl(softmax_xent_kernel<__nv_bfloat16>, grid, 256, 0, m->stream, 
          m->logits, C, (long long)m->batch * C, nullptr, m->batch, C, static_cast<__nv_bfloat16*>(m->dz[0]), ldz(m, m->L),
          (long long)m->batch * m->maxw, m->loss_part, m->sp));
    else
      NN_CUDA(launch_pdl(softmax_xent_kernel<float>, grid, 256, 0, m->stream, m->logits, C, (long long)m->batch * C, nullptr,
                                                              m->batch, C, static_cast<float*>(m->dz[0]), ldz(m, m->L),
                                                              (long long)m->batch * m->maxw, m->loss_part, m->sp));
    NN_CUDA(launch_pdl(loss_mean_kernel, m->kl, 256, 0, m->stream, m->loss_part, m->batch, m->loss));
    m->launches += 2;
  }
  // BP L..1 with the optimizer fused per layer; a masked layer's average
  // starts on the side stream as soon as its update is done
  int cur = 0;
  bool any = false;
  std::vector<cudaEvent_t>& ev_upd = capturing ? m->gev_upd : m->ev_upd;
  std::vector<cudaEvent_t>& ev_sync = capturing ? m->gev_sync : m->ev_sync;
  // one layer's sync on the side stream (+ the throttled link's busy time)
  auto sync_layer = [&](int l) -> dsx_status {
    if (hybrid) {
      any = true;
      return DSX_OK;
    }
    if (m->instrument && !any) NN_CUDA(cudaEventRecord(m->ev[7], m->side));
    NN_TRY(side_sync(m, l));
    NN_CUDA(cudaEventRecord(ev_sync[l], m->side));
    any = true;
    return DSX_OK;
  };
  for (int l = m->L - 1; l >= 0; --l) {
    NN_TRY(backward_layer(m, l, m->dz[cur], m->dz[cur ^ 1], o, m->sp));
    cur ^= 1;
    const bool sync_l = mask[l + 1] != 0 && m->K > 1;
    m->synced_prev[l] = sync_l ? 1 : 0;
    if (sync_l && m->overlap) {
      if (hybrid) {
        NN_CUDA(cudaEventRecordWithFlags(m->hev_upd[l], m->stream, cudaEventRecordExternal));
      } else {
        NN_CUDA(cudaEventRecord(ev_upd[l], m->stream));
        NN_CUDA(cudaStreamWaitEvent(m->side, ev_upd[l], 0));
      }
      NN_TRY(sync_layer(l));
    }
  }
  if (!m->overlap) {
    // ssgd / flsgd: the transfers start after the whole local step
    if (hybrid) {
      NN_CUDA(cudaEventRecordWithFlags(m->hev_upd[0], m->stream, cudaEventRecordExternal));
    } else {
      NN_CUDA(cudaEventRecord(ev_upd[0], m->stream));
      NN_CUDA(cudaStreamWaitEvent(m->side, ev_upd[0], 0));
    }
    for (int l = m->L - 1; l >= 0; --l)
      if (m->synced_prev[l]) NN_TRY(sync_layer(l));
  }
  m->any_synced = any && !capturing;
  m->side_used = any;
  if (m->instrument) {
    NN_CUDA(cudaEventRecord(m->iev[1], m->stream));
    NN_CUDA(cudaEventRecord(m->iev[2], m->side));
  }
  NN_CUDA(cudaGetLastError());
  return DSX_OK;
}

// After a hybrid graph launch: the scheduled layers' averages on the side
// stream, each behind its layer's external event record (backward order, as
// step_impl issues them eagerly), then joined into the compute stream.
dsx_status issue_hybrid_syncs(dsx_mlp* m, const unsigned char* mask) {
  bool any = false;
  if (m->overlap) {
    for (int l = m->L - 1; l >= 0; --l) {
      if (!(mask[l + 1] != 0 && m->K > 1)) continue;
      NN_CUDA(cudaStreamWaitEvent(m->side, m->hev_upd[l], 0));
      NN_TRY(side_sync(m, l));
      any = true;
    }
  } else {
    for (int l = m->L - 1; l >= 0; --l) {
      if (!(mask[l + 1] != 0 && m->K > 1)) continue;
      if (!any) NN_CUDA(cudaStreamWaitEvent(m->side, m->hev_upd[0], 0));
      NN_TRY(side_sync(m, l));
      any = true;
    }
  }
  if (any) {
    NN_CUDA(cudaEventRecord(m->ev_join, m->side));
    NN_CUDA(cudaStreamWaitEvent(m->stream, m->ev_join, 0));
  }
  NN_CUDA(cudaGetLastError());
  return DSX_OK;
}

}  // namespace
}  // namespace dsx_nn

extern "C" {

dsx_status dsx_mlp_create(const dsx_mlp_desc* d, dsx_mlp** out) {
  if (!d || !out) return nfail(DSX_ERR_ARGUMENT, "null argument");
  *out = nullptr;
  if (d->layers < 1 || !d->widths) return nfail(DSX_ERR_ARGUMENT, "layers must be >= 1");
  if (d->dtype != DSX_F32 && d->dtype != DSX_BF16) return nfail(DSX_ERR_ARGUMENT, "dtype must be DSX_F32 or DSX_BF16");
  if (d->workers_total < 1 || d->workers_local < 1 || d->worker_begin < 0 ||
      d->worker_begin + d->workers_local > d->workers_total)
    return nfail(DSX_ERR_ARGUMENT, "bad worker range");
  if (d->workers_local != 1 && d->workers_local != 2 && d->workers_local != 4 && d->workers_local != 8)
    return nfail(DSX_ERR_ARGUMENT, "workers_local must be 1, 2, 4 or 8");
  if (d->batch < 1) return nfail(DSX_ERR_ARGUMENT, "batch must be >= 1");
  if (d->optimizer < DSX_OPT_SGD || d->optimizer > DSX_OPT_ADAM) return nfail(DSX_ERR_ARGUMENT, "bad optimizer");
  for (int l = 0; l <= d->layers; ++l)
    if (d->widths[l] < 1) return nfail(DSX_ERR_ARGUMENT, "widths must be >= 1");
  if (d->dtype == DSX_BF16) {
    for (int l = 0; l < d->layers; ++l)
      if (d->widths[l] % 8)
        return nfail(DSX_ERR_ARGUMENT, "bf16 mode: input and hidden widths must be multiples of 8 (16-B rows)");
    if (d->batch % 8) return nfail(DSX_ERR_ARGUMENT, "bf16 mode: batch must be a multiple of 8");
  }
  int ndev = 0;
  NN_CUDA(cudaGetDeviceCount(&ndev));
  if (d->device < 0 || d->device >= ndev) return nfail(DSX_ERR_CUDA, "no such CUDA device");
  NN_CUDA(cudaSetDevice(d->device));
  auto* m = new dsx_mlp();
  auto cleanup = [&](dsx_status s) {
    dsx_mlp_destroy(m);
    return s;
  };
  m->device = d->device;
  m->bf16 = d->dtype == DSX_BF16;
  m->K = d->workers_total;
  m->kbegin = d->worker_begin;
  m->kl = d->workers_local;
  m->L = d->layers;
  m->widths.assign(d->widths, d->widths + d->layers + 1);
  m->batch = d->batch;
  m->opt = d->optimizer;
  m->mu = (float)d->momentum;
  m->b1 = (float)d->beta1;
  m->b2 = (float)d->beta2;
  m->eps = (float)d->eps;
  m->wd = (float)d->weight_decay;
  cudaDeviceGetAttribute(&m->nsm, cudaDevAttrMultiProcessorCount, d->device);
  long long o = 0, po = 0;
  m->packed.push_back(0);
  for (int l = 0; l < m->L; ++l) {
    const long long in = m->widths[l], outw = m->widths[l + 1];
    m->off.push_back(o);
    m->boff.push_back(o + in * outw);
    o = (o + in * outw + outw + 63) / 64 * 64;
    po += in * outw + outw;
    m->packed.push_back(po);
  }
  m->P = o;
  m->maxw = *std::max_element(m->widths.begin(), m->widths.end());
  m->maxw = (m->maxw + 7) / 8 * 8;
  const size_t arena = 4ull * m->P * m->kl;
  auto alloc = [&](void** p, size_t bytes) -> bool {
    if (cudaMalloc(p, bytes) != cudaSuccess) return false;
    cudaMemset(*p, 0, bytes);
    return true;
  };
  if (!alloc((void**)&m->params, arena) || !alloc((void**)&m->grads, arena) ||
      (m->opt != DSX_OPT_SGD && !alloc((void**)&m->mom, arena)) ||
      (m->opt == DSX_OPT_ADAM && !alloc((void**)&m->var, arena)) ||
      (m->bf16 && !alloc((void**)&m->pbf, 2ull * m->P * m->kl)))
    return cleanup(nfail(DSX_ERR_CUDA, "cudaMalloc(parameter arenas) failed"));
  m->act.assign(m->L, nullptr);
  for (int l = 0; l < m->L; ++l)
    if (!alloc(&m->act[l], esz(m) * m->kl * (size_t)m->batch * m->widths[l]))
      return cleanup(nfail(DSX_ERR_CUDA, "cudaMalloc(activations) failed"));
  for (auto& p : m->dz)
    if (!alloc(&p, esz(m) * m->kl * (size_t)m->batch * m->maxw))
      return cleanup(nfail(DSX_ERR_CUDA, "cudaMalloc(gradients) failed"));
  if (!alloc((void**)&m->logits, 4ull * m->kl * m->batch * m->widths[m->L]) ||
      !alloc((void**)&m->xin, 4ull * m->kl * m->batch * m->widths[0]) ||
      !alloc((void**)&m->labels, 4ull * m->kl * m->batch) || !alloc((void**)&m->loss_part, 4ull * m->kl * m->batch) ||
      !alloc((void**)&m->loss, 4ull * m->kl))
    return cleanup(nfail(DSX_ERR_CUDA, "cudaMalloc(io) failed"));
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if (cudaStreamCreateWithPriority(&m->stream, cudaStreamNonBlocking, lo) != cudaSuccess ||
      cudaStreamCreateWithPriority(&m->side, cudaStreamNonBlocking, hi) != cudaSuccess)
    return cleanup(nfail(DSX_ERR_CUDA, "stream creation failed"));
  m->ev_upd.assign(m->L, nullptr);
  m->ev_sync.assign(m->L, nullptr);
  for (int l = 0; l < m->L; ++l) {
    cudaEventCreateWithFlags(&m->ev_upd[l], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&m->ev_sync[l], cudaEventDisableTiming);
  }
  for (auto& e : m->ev) cudaEventCreate(&e);
  for (auto& e : m->iev) cudaEventCreate(&e);
  m->synced_prev.assign(m->L, 0);
  cudaEventCreateWithFlags(&m->ev_join, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&m->ev_drain, cudaEventDisableTiming);
  m->gev_upd.assign(m->L, nullptr);
  m->gev_sync.assign(m->L, nullptr);
  m->hev_upd.assign(m->L, nullptr);
  for (auto& e : m->hev_upd) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  for (int l = 0; l < m->L; ++l) {
    cudaEventCreateWithFlags(&m->gev_upd[l], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&m->gev_sync[l], cudaEventDisableTiming);
  }
  m->ring_ev.assign(64, nullptr);
  for (auto& e : m->ring_ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  if (cudaMalloc(&m->sp, sizeof(StepDev)) != cudaSuccess ||
      cudaHostAlloc(&m->ring, sizeof(StepDev) * m->ring_ev.size(), cudaHostAllocDefault) != cudaSuccess)
    return cleanup(nfail(DSX_ERR_CUDA, "step-parameter buffers"));
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cleanup(nfail(DSX_ERR_CUDA, std::string("mlp init: ") + cudaGetErrorString(e)));
  *out = m;
  return DSX_OK;
}

dsx_status dsx_mlp_destroy(dsx_mlp* m) {
  if (!m) return DSX_OK;
  cudaSetDevice(m->device);
  if (m->stream) cudaStreamSynchronize(m->stream);
  if (m->side) cudaStreamSynchronize(m->side);
  if (m->comm) ncclCommDestroy(m->comm);
  for (void* p : {(void*)m->params, (void*)m->pbf, (void*)m->grads, (void*)m->mom, (void*)m->var, (void*)m->logits,
                  (void*)m->xin, (void*)m->labels, (void*)m->loss_part, (void*)m->loss, m->dz[0], m->dz[1]})
    if (p) cudaFree(p);
  for (void* p : m->act)
    if (p) cudaFree(p);
  for (auto e : m->ev_upd)
    if (e) cudaEventDestroy(e);
  for (auto e : m->ev_sync)
    if (e) cudaEventDestroy(e);
  for (auto e : m->ev)
    if (e) cudaEventDestroy(e);
  for (auto e : m->iev)
    if (e) cudaEventDestroy(e);
  for (auto& kv : m->graph_cache) cudaGraphExecDestroy(kv.second.exec);
  for (auto e : m->ring_ev)
    if (e) cudaEventDestroy(e);
  if (m->ev_join) cudaEventDestroy(m->ev_join);
  if (m->ev_drain) cudaEventDestroy(m->ev_drain);
  for (auto e : m->hev_upd)
    if (e) cudaEventDestroy(e);
  for (auto e : m->gev_upd)
    if (e) cudaEventDestroy(e);
  for (auto e : m->gev_sync)
    if (e) cudaEventDestroy(e);
  if (m->sp) cudaFree(m->sp);
  if (m->ring) cudaFreeHost(m->ring);
  if (m->stream) cudaStreamDestroy(m->stream);
  if (m->side) cudaStreamDestroy(m->side);
  delete m;
  return DSX_OK;
}

dsx_status dsx_mlp_param_layout(dsx_mlp* m, uint64_t* total, uint64_t* offsets) {
  if (!m) return nfail(DSX_ERR_ARGUMENT, "null mlp");
  if (total) *total = (uint64_t)m->packed.back();
  if (offsets)
    for (int l = 0; l <= m->L; ++l) offsets[l] = (uint64_t)m->packed[l];
  return DSX_OK;
}

namespace {
dsx_status copy_packed(dsx_mlp* m, float* dev_arena, int local, float* host, bool to_dev) {
  for (int l = 0; l < m->L; ++l) {
    const long long n = m->packed[l + 1] - m->packed[l];
    float* d = dev_arena + (long long)local * m->P + m->off[l];
    float* h = host + m->packed[l];
    // W and b are adjacent in both layouts (b follows W immediately)
    NN_CUDA(cudaMemcpy(to_dev ? (void*)d : (void*)h, to_dev ? (void*)h : (void*)d, 4ull * n,
                       to_dev ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost));
  }
  return DSX_OK;
}
}  // namespace

dsx_status dsx_mlp_set_params(dsx_mlp* m, int local, const float* packed) {
  NN_TRY(check(m));
  if (local < 0 || local >= m->kl || !packed) return nfail(DSX_ERR_ARGUMENT, "bad local worker / null params");
  NN_CUDA(cudaStreamSynchronize(m->side));
  NN_CUDA(cudaStreamSynchronize(m->stream));
  NN_TRY(copy_packed(m, m->params, local, const_cast<float*>(packed), true));
  if (m->bf16) {
    cast_bf16_kernel<<<blocks_for(m->P, m->nsm), 256, 0, m->stream>>>(m->params + (long long)local * m->P,
                                                                     m->pbf + (long long)local * m->P, 0, 1, 0, m->P);
    NN_CUDA(cudaStreamSynchronize(m->stream));
  }
  return DSX_OK;
}

dsx_status dsx_mlp_get_params(dsx_mlp* m, int local, float* packed) {
  NN_TRY(check(m));
  if (local < 0 || local >= m->kl || !packed) return nfail(DSX_ERR_ARGUMENT, "bad local worker / null params");
  NN_CUDA(cudaStreamSynchronize(m->side));
  NN_CUDA(cudaStreamSynchronize(m->stream));
  return copy_packed(m, m->params, local, packed, false);
}

dsx_status dsx_mlp_get_state(dsx_mlp* m, int local, float* mom, float* var) {
  NN_TRY(check(m));
  if (local < 0 || local >= m->kl) return nfail(DSX_ERR_ARGUMENT, "bad local worker");
  NN_CUDA(cudaStreamSynchronize(m->stream));
  if (mom && m->mom) NN_TRY(copy_packed(m, m->mom, local, mom, false));
  if (var && m->var) NN_TRY(copy_packed(m, m->var, local, var, false));
  return DSX_OK;
}

dsx_status dsx_mlp_set_batch(dsx_mlp* m, const float* x, const int32_t* labels, int on_device) {
  NN_TRY(check(m));
  if (!x || !labels) return nfail(DSX_ERR_ARGUMENT, "null batch");
  if (on_device) {
    m->x_dev = x;
    m->labels_dev = labels;
    return DSX_OK;
  }
  const size_t nx = 4ull * m->kl * m->batch * m->widths[0], nl = 4ull * m->kl * m->batch;
  NN_CUDA(cudaMemcpyAsync(m->xin, x, nx, cudaMemcpyHostToDevice, m->stream));
  NN_CUDA(cudaMemcpyAsync(m->labels, labels, nl, cudaMemcpyHostToDevice, m->stream));
  m->x_dev = m->xin;
  m->labels_dev = m->labels;
  return DSX_OK;
}

dsx_status dsx_mlp_step(dsx_mlp* m, double lr, long long step_index, const unsigned char* mask) {
  NN_TRY(check(m));
  if (!mask) return nfail(DSX_ERR_ARGUMENT, "null mask");
  NN_TRY(write_step(m, lr, step_index));
  // graphs: one rank captures the averages too; several ranks capture the
  // compute only (hybrid) and issue the NCCL averages eagerly behind it
  if (!m->graphs || m->instrument) return step_impl(m, lr, step_index, mask, false);
  const bool hybrid = m->nranks > 1;
  // one graph per distinct mask (H of them for a partial schedule), captured
  // on first use; the averages are joined into the compute stream at the end
  const std::string key(reinterpret_cast<const char*>(mask), (size_t)m->L + 1);
  dsx_mlp::Graph* g = nullptr;
  for (auto& kv : m->graph_cache)
    if (kv.first == key) g = &kv.second;
  if (!g) {
    // a capture starts with the eager side-stream work joined in
    NN_CUDA(cudaEventRecord(m->ev_drain, m->side));
    NN_CUDA(cudaStreamWaitEvent(m->stream, m->ev_drain, 0));
    const uint64_t before = m->launches;
    NN_CUDA(cudaStreamBeginCapture(m->stream, cudaStreamCaptureModeThreadLocal));
    dsx_status st = step_impl(m, lr, step_index, mask, true, hybrid);
    if (st == DSX_OK && m->side_used && !hybrid) {  // (a mask with nothing to average never forks)
      if (cudaEventRecord(m->ev_join, m->side) != cudaSuccess ||
          cudaStreamWaitEvent(m->stream, m->ev_join, 0) != cudaSuccess)
        st = nfail(DSX_ERR_CUDA, "graph capture: joining the sync stream failed");
    }
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(m->stream, &graph);
    if (st != DSX_OK) {
      if (graph) cudaGraphDestroy(graph);
      return st;
    }
    if (ce != cudaSuccess) return nfail(DSX_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    dsx_mlp::Graph ng;
    const cudaError_t ie = cudaGraphInstantiate(&ng.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) return nfail(DSX_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ie));
    ng.launches = m->launches - before;
    m->launches = before;
    m->graph_cache.emplace_back(key, ng);
    g = &m->graph_cache.back().second;
  }
  NN_CUDA(cudaGraphLaunch(g->exec, m->stream));
  m->launches += g->launches;
  if (hybrid) NN_TRY(issue_hybrid_syncs(m, mask));
  for (int l = 0; l < m->L; ++l) m->synced_prev[l] = (mask[l + 1] != 0 && m->K > 1) ? 1 : 0;
  return DSX_OK;
}

dsx_status dsx_mlp_last_loss(dsx_mlp* m, float* loss) {
  NN_TRY(check(m));
  if (!loss) return nfail(DSX_ERR_ARGUMENT, "null out");
  NN_CUDA(cudaStreamSynchronize(m->stream));
  NN_CUDA(cudaMemcpy(loss, m->loss, 4ull * m->kl, cudaMemcpyDeviceToHost));
  return DSX_OK;
}

dsx_status dsx_mlp_sync(dsx_mlp* m) {
  NN_TRY(check(m));
  NN_CUDA(cudaStreamSynchronize(m->side));
  NN_CUDA(cudaStreamSynchronize(m->stream));
  NN_CUDA(cudaGetLastError());
  return DSX_OK;
}

dsx_status dsx_mlp_comm_init(dsx_mlp* m, const unsigned char id[128], int nranks, int rank) {
  NN_TRY(check(m));
  if (!id || nranks < 1 || rank < 0 || rank >= nranks) return nfail(DSX_ERR_ARGUMENT, "bad comm args");
  if (m->comm) return nfail(DSX_ERR_STATE, "comm already initialised");
  if (m->K != m->kl * nranks || m->kbegin != rank * m->kl)
    return nfail(DSX_ERR_ARGUMENT, "ranks must hold equal contiguous worker ranges");
  ncclUniqueId u;
  std::memcpy(u.internal, id, 128);
  NN_NCCL(ncclCommInitRank(&m->comm, nranks, u, rank));
  m->nranks = nranks;
  m->rank = rank;
  return DSX_OK;
}

dsx_status dsx_mlp_set_instrument(dsx_mlp* m, int enabled) {
  NN_TRY(check(m));
  m->instrument = enabled != 0;
  return DSX_OK;
}

dsx_status dsx_mlp_last_step_times(dsx_mlp* m, float* out4) {
  NN_TRY(check(m));
  if (!out4) return nfail(DSX_ERR_ARGUMENT, "null out");
  if (!m->instrument) return nfail(DSX_ERR_STATE, "instrumentation is off");
  // step end = max(compute done, sync done): record on the compute stream
  // after it waited for the side stream
  NN_CUDA(cudaStreamWaitEvent(m->stream, m->iev[2], 0));
  NN_CUDA(cudaEventRecord(m->iev[3], m->stream));
  NN_CUDA(cudaEventSynchronize(m->iev[3]));
  float total = 0, comp = 0, span = 0, done = 0;
  NN_CUDA(cudaEventElapsedTime(&total, m->iev[0], m->iev[3]));
  NN_CUDA(cudaEventElapsedTime(&comp, m->iev[0], m->iev[1]));
  if (m->any_synced) {
    NN_CUDA(cudaEventElapsedTime(&span, m->ev[7], m->iev[2]));
    NN_CUDA(cudaEventElapsedTime(&done, m->iev[0], m->iev[2]));
  }
  out4[0] = total;
  out4[1] = comp;
  out4[2] = m->any_synced ? span : 0.f;
  out4[3] = m->any_synced ? std::max(0.f, done - comp) : 0.f;
  return DSX_OK;
}

dsx_status dsx_mlp_profile(dsx_mlp* m, int reps, double* t_fp, double* t_bp, double* t_comm) {
  NN_TRY(check(m));
  if (!t_fp || !t_bp || !t_comm) return nfail(DSX_ERR_ARGUMENT, "null out");
  if (!m->x_dev) return nfail(DSX_ERR_STATE, "profile needs a batch (dsx_mlp_set_batch)");
  reps = std::max(1, reps);
  NN_TRY(write_step(m, 0.0, 0));
  NN_CUDA(cudaStreamSynchronize(m->side));
  NN_CUDA(cudaStreamSynchronize(m->stream));
  // the profile must not change the state: snapshot params / states
  std::vector<void*> keep;
  auto snap = [&](void* p, size_t bytes) -> dsx_status {
    void* c = nullptr;
    if (!p) {
      keep.push_back(nullptr);
      return DSX_OK;
    }
    NN_CUDA(cudaMalloc(&c, bytes));
    NN_CUDA(cudaMemcpy(c, p, bytes, cudaMemcpyDeviceToDevice));
    keep.push_back(c);
    return DSX_OK;
  };
  const size_t arena = 4ull * m->P * m->kl;
  NN_TRY(snap(m->params, arena));
  NN_TRY(snap(m->mom, arena));
  NN_TRY(snap(m->var, arena));
  std::vector<cudaEvent_t> e(2 * m->L + 2);
  for (auto& x : e) NN_CUDA(cudaEventCreate(&x));
  std::vector<std::vector<float>> fp(m->L), bp(m->L), cm(m->L);
  OptArgs o{};
  o.kind = m->opt;
  o.lr = 0.f;
  o.mu = m->mu;
  o.b1 = m->b1;
  o.b2 = m->b2;
  o.eps = m->eps;
  o.bc1 = o.bc2 = 1.f;
  for (int r = 0; r < reps + 1; ++r) {
    NN_TRY(prepare_input(m));
    NN_CUDA(cudaEventRecord(e[0], m->stream));
    for (int l = 0; l < m->L; ++l) {
      NN_TRY(forward_layer(m, l));
      NN_CUDA(cudaEventRecord(e[l + 1], m->stream));
    }
    const int C = m->widths[m->L];
    dim3 grid((m->batch * 32 + 255) / 256, m->kl);
    if (m->bf16)
      NN_CUDA(launch_pdl(softmax_xent_kernel<__nv_bfloat16>, grid, 256, 0, m->stream, 
          m->logits, C, (long long)m->batch * C, nullptr, m->batch, C, static_cast<__nv_bfloat16*>(m->dz[0]), ldz(m, m->L),
          (long long)m->batch * m->maxw, m->loss_part, m->sp));
    else
      NN_CUDA(launch_pdl(softmax_xent_kernel<float>, grid, 256, 0, m->stream, m->logits, C, (long long)m->batch * C, nullptr,
                                                              m->batch, C, static_cast<float*>(m->dz[0]), ldz(m, m->L),
                                                              (long long)m->batch * m->maxw, m->loss_part, m->sp));
    NN_CUDA(cudaEventRecord(e[m->L + 1], m->stream));
    int cur = 0;
    for (int l = m->L - 1; l >= 0; --l) {
      NN_TRY(backward_layer(m, l, m->dz[cur], m->dz[cur ^ 1], o, nullptr));
      cur ^= 1;
      NN_CUDA(cudaEventRecord(e[m->L + 1 + (m->L - l)], m->stream));
    }
    NN_CUDA(cudaStreamSynchronize(m->stream));
    if (r == 0) continue;  // warm-up
    for (int l = 0; l < m->L; ++l) {
      float t = 0;
      NN_CUDA(cudaEventElapsedTime(&t, e[l], e[l + 1]));
      fp[l].push_back(t);
      // BP of layer l ends at e[L+1+(L-l)], starts at the previous event
      NN_CUDA(cudaEventElapsedTime(&t, e[m->L + (m->L - l)], e[m->L + 1 + (m->L - l)]));
      bp[l].push_back(t);
    }
  }
  // the average of each layer alone (side stream)
  for (int r = 0; r < reps + 1 && m->K > 1; ++r) {
    for (int l = 0; l < m->L; ++l) {
      NN_CUDA(cudaEventRecord(e[0], m->side));
      NN_TRY(average_layer(m, l, m->side));
      NN_CUDA(cudaEventRecord(e[1], m->side));
      NN_CUDA(cudaEventSynchronize(e[1]));
      float t = 0;
      NN_CUDA(cudaEventElapsedTime(&t, e[0], e[1]));
      if (r > 0) cm[l].push_back(t);
    }
  }
  auto med = [](std::vector<float> v) {
    if (v.empty()) return 0.0;
    std::sort(v.begin(), v.end());
    return (double)v[v.size() / 2] * 1e-3;
  };
  for (int l = 0; l < m->L; ++l) {
    t_fp[l] = med(fp[l]);
    t_bp[l] = med(bp[l]);
    t_comm[l] = med(cm[l]);
  }
  for (auto x : e) cudaEventDestroy(x);
  // restore
  void* live[3] = {m->params, m->mom, m->var};
  for (int i = 0; i < 3; ++i)
    if (keep[i]) {
      NN_CUDA(cudaMemcpy(live[i], keep[i], arena, cudaMemcpyDeviceToDevice));
      cudaFree(keep[i]);
    }
  if (m->bf16) {
    cast_bf16_kernel<<<blocks_for(m->P * m->kl, m->nsm), 256, 0, m->stream>>>(m->params, m->pbf, 0, 1, 0,
                                                                             m->P * (long long)m->kl);
    NN_CUDA(cudaStreamSynchronize(m->stream));
  }
  return DSX_OK;
}

dsx_status dsx_mlp_event_record(dsx_mlp* m, int slot) {
  NN_TRY(check(m));
  if (slot < 0 || slot >= 7) return nfail(DSX_ERR_ARGUMENT, "slot must be in [0, 7)");
  // include pending averages on the side stream
  NN_CUDA(cudaEventRecord(m->iev[2], m->side));
  NN_CUDA(cudaStreamWaitEvent(m->stream, m->iev[2], 0));
  NN_CUDA(cudaEventRecord(m->ev[slot], m->stream));
  return DSX_OK;
}

dsx_status dsx_mlp_event_elapsed(dsx_mlp* m, int a, int b, float* ms) {
  NN_TRY(check(m));
  if (!ms || a < 0 || a >= 7 || b < 0 || b >= 7) return nfail(DSX_ERR_ARGUMENT, "bad slots");
  NN_CUDA(cudaEventSynchronize(m->ev[b]));
  NN_CUDA(cudaEventElapsedTime(ms, m->ev[a], m->ev[b]));
  return DSX_OK;
}

dsx_status dsx_mlp_launch_count(dsx_mlp* m, uint64_t* out) {
  if (!m || !out) return nfail(DSX_ERR_ARGUMENT, "null argument");
  *out = m->launches;
  return DSX_OK;
}

dsx_status dsx_mlp_set_link(dsx_mlp* m, double bandwidth, double latency) {
  NN_TRY(check(m));
  if (!(latency >= 0.0)) return nfail(DSX_ERR_ARGUMENT, "latency must be >= 0");
  m->link_bw = bandwidth > 0.0 ? bandwidth : 0.0;
  m->link_lat = latency;
  return dsx_mlp_set_graphs(m, m->graphs ? 1 : 0);
}

dsx_status dsx_mlp_set_overlap(dsx_mlp* m, int enabled) {
  NN_TRY(check(m));
  m->overlap = enabled != 0;
  return dsx_mlp_set_graphs(m, m->graphs ? 1 : 0);
}

dsx_status dsx_mlp_set_graphs(dsx_mlp* m, int enabled) {
  NN_TRY(check(m));
  NN_CUDA(cudaStreamSynchronize(m->stream));
  NN_CUDA(cudaStreamSynchronize(m->side));
  for (auto& kv : m->graph_cache) cudaGraphExecDestroy(kv.second.exec);
  m->graph_cache.clear();  // link / overlap settings are baked into a graph
  m->graphs = enabled != 0;
  return DSX_OK;
}

}  // extern "C"
