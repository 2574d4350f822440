/*
 * dsx_nn.h — C ABI of the NN local step: a K-worker MLP trained with
 * DreamDDP's layer-wise scheduled partial synchronization on sm_100a.
 *
 * The reference has no neural network: its workers
 * are quadratic-lab parameter vectors.  BASELINE.json configs[0] asks for a
 * "small MLP on synthetic data, 4 workers, H=4, partial layer-wise sync", and
 * north_star (1) for the per-worker local step as forward/backward of the
 * layer stack plus the fused SGD-momentum/Adam update on hand-written
 * kernels (tcgen05/TMA for the dense GEMMs).  This ABI is that step, shaped
 * like the reference's trainer entry points so the same scheduler drives it:
 *   dsx_mlp_create   model + layer registration: registered layer l (1-based,
 *                    l = 1 the input side, as in profile.hpp:31-64) is Linear
 *                    layer l, its parameters W_l[out][in] then b_l[out] one
 *                    contiguous range of the worker's arena (a sync set is a
 *                    byte range, as trainer.cpp:50-56 lays out blocks).
 *   dsx_mlp_step     plsgd_step (trainer.cpp:187-235) with the quadratic's
 *                    gradient replaced by FP + softmax cross-entropy + BP and
 *                    the SGD update by the layer's optimizer; after BP(l) and
 *                    update(l) the masked layer l is averaged over all K
 *                    workers on a high-priority side stream (Alg. 1,
 *                    parameters only, optimizer states stay
 *                    local), overlapping BP(l-1..1).  mask is the reference's
 *                    1-based vector<bool> (trainer.cpp:202-224).
 *   dsx_mlp_profile  CUDA-event per-layer FP / BP / sync times, the input of
 *                    write_profile -> schedule_dfs (profile.cpp:160-174).
 * Plain pointers and sizes only; every call returns a dsx_status and
 * the last-error string of dsx.h holds the message.
 */
#ifndef DREAMDDP_DSX_NN_H_
#define DREAMDDP_DSX_NN_H_

#include <stddef.h>
#include <stdint.h>

#include "dsx.h"

#ifdef __cplusplus
extern "C" {
#endif

/* GEMM / activation arithmetic (DSX_F32 = 1 as in dsx.h) */
enum { DSX_BF16 = 2 };

/* optimizers (states are per worker and never synchronized) */
enum { DSX_OPT_SGD = 0, DSX_OPT_MOMENTUM = 1, DSX_OPT_ADAM = 2 };

/* ---- GEMM test hook: C[b][m][n] = epi(sum_k A(m,k) B(n,k)) ------------- */
enum { DSX_EPI_F32 = 0, DSX_EPI_BIAS_ACT = 1, DSX_EPI_DRELU = 2, DSX_EPI_ADD = 3,
       DSX_EPI_BIAS_ADD_ACT = 4 /* act(acc + bias + mask) */, DSX_EPI_ADD_DRELU = 5 /* (acc + mask) * (mask2 > 0) */ };
typedef struct dsx_gemm_desc {
  int dtype;                 /* DSX_BF16: tcgen05 kernel, DSX_F32: SIMT kernel */
  int M, N, K, batch;
  int a_mn, b_mn;            /* 0: K-major (A[m*lda+k]), 1: MN-major (A[k*lda+m]) */
  const void* A;
  long long lda, strideA;    /* elements */
  const void* B;
  long long ldb, strideB;
  void* C;
  long long ldc, strideC;
  int out_dtype;             /* DSX_F32 or DSX_BF16 (epi != DSX_EPI_F32) */
  int epi, relu, accumulate;
  const float* bias;
  long long strideBias;
  const void* mask;          /* DSX_EPI_DRELU: element (m,n) > 0 keeps the gradient */
  long long ldmask, strideMask;
  int bn;                    /* tensor-core tile width 64/128/256 (0: auto) */
  void* stream;              /* cudaStream_t (NULL: default stream) */
  int ksplit;                /* split-K (bf16, DSX_EPI_F32, no accumulate): split s of K writes */
  long long strideSplit;     /* its partial at C + s * strideSplit; 0/1: off */
  /* implicit-GEMM 3x3 / stride 1 / pad 1 convolution (bf16; M, N, K derived):
   * conv = 1 forward (A = x NHWC, B = W[o][kh][kw][c]), 2 wgrad (A = dy,
   * B = x), 3 dgrad (A = dy, B = W); strideA / strideB are per batch entry;
   * 0: plain GEMM */
  int conv, conv_h, conv_w, conv_images, conv_cin, conv_cout;  /* conv_h / conv_w: input grid */
  int conv_stride, conv_k;   /* 0 -> 1 / 3; stride 2 (3x3 or 1x1): forward and wgrad */
  const void* mask2;         /* DSX_EPI_ADD_DRELU: the ReLU' operand (mask is the addend) */
  long long ldmask2, strideMask2;
} dsx_gemm_desc;
dsx_status dsx_gemm(const dsx_gemm_desc* d);

/* ---- the K-worker MLP ------------------------------------------------- */
typedef struct dsx_mlp dsx_mlp;
typedef struct dsx_mlp_desc {
  int device;
  int dtype;                 /* DSX_F32 (fp32 SIMT GEMMs, parity) | DSX_BF16 (tcgen05) */
  int workers_total;         /* K */
  int worker_begin;          /* global id of the first local worker */
  int workers_local;
  int layers;                /* L Linear layers; ReLU between them */
  const int* widths;         /* [layers + 1]: input, hidden..., classes */
  int batch;                 /* samples per worker per step */
  int optimizer;             /* DSX_OPT_* */
  double momentum;           /* SGD momentum (PyTorch semantics: v = mu v + g) */
  double beta1, beta2, eps;  /* Adam */
  double weight_decay;       /* L2 added to the gradient (SGD) / decoupled (Adam: AdamW) */
} dsx_mlp_desc;

dsx_status dsx_mlp_create(const dsx_mlp_desc* desc, dsx_mlp** out);
dsx_status dsx_mlp_destroy(dsx_mlp* m);
/* Per-worker parameter count and the packed host layout: layer l (1..L)
 * occupies [offsets[l-1], offsets[l]) = W_l[out][in] row-major, then b_l. */
dsx_status dsx_mlp_param_layout(dsx_mlp* m, uint64_t* total, uint64_t* offsets /* [layers+1] */);
dsx_status dsx_mlp_set_params(dsx_mlp* m, int local, const float* packed);
dsx_status dsx_mlp_get_params(dsx_mlp* m, int local, float* packed);
/* Optimizer states (packed like the parameters; v only for Adam). */
dsx_status dsx_mlp_get_state(dsx_mlp* m, int local, float* mom, float* var);
/* The next step's data: x[workers_local][batch][in] fp32, labels
 * [workers_local][batch] int32, host or device pointers (on_device).  Host
 * data is copied on the compute stream (the e2e path); device data is used
 * in place (must stay valid until the step ran). */
dsx_status dsx_mlp_set_batch(dsx_mlp* m, const float* x, const int32_t* labels, int on_device);
/* One iteration: FP, loss, BP with the fused optimizer per layer, scheduled
 * averaging of the masked layers (mask[layers+1], 1-based).  lr is the
 * step's learning rate; step_index (0-based) drives Adam's bias correction.
 * Asynchronous. */
dsx_status dsx_mlp_step(dsx_mlp* m, double lr, long long step_index, const unsigned char* mask);
/* Mean cross-entropy of each local worker's last batch (synchronizes). */
dsx_status dsx_mlp_last_loss(dsx_mlp* m, float* loss /* [workers_local] */);
dsx_status dsx_mlp_sync(dsx_mlp* m);
/* Multi-GPU: one rank per GPU, id = ncclUniqueId from rank 0 (dsx.h). */
dsx_status dsx_mlp_comm_init(dsx_mlp* m, const unsigned char id[128], int nranks, int rank);
/* Per-step CUDA-event instrumentation: out4 = ms of [whole step, local
 * compute (FP+BP+updates), sync span, exposed sync = max(0, last sync done -
 * local compute done)] of the last step. */
dsx_status dsx_mlp_set_instrument(dsx_mlp* m, int enabled);
dsx_status dsx_mlp_last_step_times(dsx_mlp* m, float* out4);
/* CUDA-event layer profiler: t_fp[l], t_bp[l] (BP incl. the optimizer
 * update), t_comm[l] (cross-worker average of the layer alone; 0 with one
 * worker) in seconds, median of reps. */
dsx_status dsx_mlp_profile(dsx_mlp* m, int reps, double* t_fp, double* t_bp, double* t_comm);
/* Timing on the compute stream (slots 0..7). */
dsx_status dsx_mlp_event_record(dsx_mlp* m, int slot);
dsx_status dsx_mlp_event_elapsed(dsx_mlp* m, int from_slot, int to_slot, float* ms);
dsx_status dsx_mlp_launch_count(dsx_mlp* m, uint64_t* out);
/* Throttled link (the paper's low-bandwidth regime): every synced layer
 * additionally occupies the FIFO sync stream for latency + layer_bytes /
 * bandwidth seconds (comm_time, profile.cpp:103-110).  bandwidth <= 0: off. */
dsx_status dsx_mlp_set_link(dsx_mlp* m, double bandwidth, double latency);
/* enabled (default): a layer's average starts as soon as its BP + update is
 * done (wfbp / plsgd); 0: all averages after the whole local step (the ssgd
 * and flsgd modes). */
dsx_status dsx_mlp_set_overlap(dsx_mlp* m, int enabled);
/* Replay the step from CUDA graphs: one captured per distinct sync mask on
 * first use (the step's lr / bias corrections / batch pointers are read from
 * device memory, so every step replays the same graph), the sync stream's
 * averages joined at the end of each.  With several ranks the graph holds
 * the compute only (external event records where each scheduled layer's
 * update ends) and the NCCL averages are enqueued eagerly behind those
 * events after every launch.  0 disables (default). */
dsx_status dsx_mlp_set_graphs(dsx_mlp* m, int enabled);

/* ---- conv stack: BASELINE configs[1] (ResNet-18 shape) as a network ----
 * CIFAR ResNet-18 geometry without normalisation layers: 3x3 stem (in_channels
 * zero-padded to 8) -> 4 stages x 2 basic blocks of widths width<<s (stride 2
 * and a 1x1 projection shortcut entering stages 1-3) -> global average pool ->
 * linear head.  Registered layers (1-based, forward order): the stem, per
 * block conv a, conv b, [shortcut], then the head (21 for ResNet-18); layer
 * l's packed parameters are W_l [Cout][kh][kw][Cin] then b_l [Cout].  BP
 * runs a block's shortcut, b, a; each layer's optimizer runs right after its
 * gradients and a scheduled layer's average starts on the side stream — the
 * same step semantics as dsx_mlp_step. */
typedef struct dsx_cnn dsx_cnn;
typedef struct dsx_cnn_desc {
  int device;
  int dtype;                 /* DSX_F32 (SIMT, parity) | DSX_BF16 (tcgen05) */
  int workers_total, worker_begin, workers_local;  /* workers_local in {1,2,4,8} */
  int width;                 /* stem width (ResNet-18: 64), multiple of 8 */
  int image;                 /* square input side (32), multiple of 8 */
  int in_channels;           /* 1..8 (3) */
  int classes;               /* head outputs (10) */
  int batch;                 /* per-worker batch */
  int optimizer;             /* DSX_OPT_* */
  double momentum, beta1, beta2, eps, weight_decay;
} dsx_cnn_desc;

dsx_status dsx_cnn_create(const dsx_cnn_desc* desc, dsx_cnn** out);
dsx_status dsx_cnn_destroy(dsx_cnn* m);
/* layers, packed total and offsets [layers+1], fan-in per layer (k*k*Cin) */
dsx_status dsx_cnn_param_layout(dsx_cnn* m, int* layers, uint64_t* total, uint64_t* offsets, int* fan_in);
dsx_status dsx_cnn_set_params(dsx_cnn* m, int local, const float* packed);
dsx_status dsx_cnn_get_params(dsx_cnn* m, int local, float* packed);
/* x: fp32 NHWC [workers_local][batch][image][image][in_channels], labels
 * int32 [workers_local][batch]; on_device as in dsx_mlp_set_batch */
dsx_status dsx_cnn_set_batch(dsx_cnn* m, const float* x, const int32_t* labels, int on_device);
dsx_status dsx_cnn_step(dsx_cnn* m, double lr, long long step_index, const unsigned char* mask);
dsx_status dsx_cnn_last_loss(dsx_cnn* m, float* loss /* [workers_local] */);
dsx_status dsx_cnn_sync(dsx_cnn* m);
dsx_status dsx_cnn_comm_init(dsx_cnn* m, const unsigned char id[128], int nranks, int rank);
dsx_status dsx_cnn_set_instrument(dsx_cnn* m, int enabled);
dsx_status dsx_cnn_last_step_times(dsx_cnn* m, float* out4);
dsx_status dsx_cnn_event_record(dsx_cnn* m, int slot);
dsx_status dsx_cnn_event_elapsed(dsx_cnn* m, int from_slot, int to_slot, float* ms);
/* CUDA-event per-layer FP / BP (+ update) / average times in seconds (median
 * of reps lr-0 steps; parameters and optimizer states restored) — the input
 * of dsc_write_profile -> the DFS scheduler, as dsx_mlp_profile. */
dsx_status dsx_cnn_profile(dsx_cnn* m, int reps, double* t_fp, double* t_bp, double* t_comm);
dsx_status dsx_cnn_launch_count(dsx_cnn* m, uint64_t* out);
/* Throttled sync link and overlap control, as dsx_mlp_set_link /
 * dsx_mlp_set_overlap (the four-mode runs of paper_2502_11058_b200/modes.py). */
dsx_status dsx_cnn_set_link(dsx_cnn* m, double bandwidth, double latency);
dsx_status dsx_cnn_set_overlap(dsx_cnn* m, int enabled);

#ifdef __cplusplus
}
#endif

#endif /* DREAMDDP_DSX_NN_H_ */
