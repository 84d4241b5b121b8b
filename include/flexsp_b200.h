/*
 * flexsp_b200.h — C-ABI of the B200-native FlexSP sequence-parallel step.
 *
 * The reference (seqplan, /root/reference/pkg) stops at the Plan object that
 * "the executor sequentially reads one plan per iteration to train"
 * (pkg/src/seqplan/domain.py:332-400).  It has no executor and
 * therefore no FFI of its own: its boundary is the Python/JSON Plan
 * (GroupDispatch.sequence_indices, domain.py:332-342; plan JSON schema 1,
 * domain.py:390-397, pkg/docs/formats.md:74-105).  The entry points below are
 * what that executor binds (see INTEGRATION.md for the ctypes stub); each
 * replaces one step of the paper's executor:
 *
 *   fsp_pack_rows / fsp_unpack_rows  — "scatters the data into the corresponding
 *        group" + sequence packing
 *   fsp_a2a_seq2head / fsp_a2a_head2seq / fsp_group_barrier — Ulysses AlltoAll,
 *        Eq. (2) and Eq. (4), NCCL in the paper
 *   fsp_attn_fwd / fsp_attn_bwd — Eq. (3) through flash-attn varlen
 *        in the paper
 *
 * Conventions (mirroring the reference's error/ownership rules, domain.py:17-34):
 *   - every buffer is allocated by the caller; the library never allocates
 *     device memory and keeps no state except a cached driver entry point;
 *   - all pointers named d_* / tensors are device pointers, *_host are host;
 *   - `stream` is a cudaStream_t passed as void*;
 *   - return 0 on success; FSP_ERR_INVALID for a bad argument/layout (the analog
 *     of seqplan.ValidationError, Python maps it to ValueError); FSP_ERR_CUDA for a
 *     CUDA failure (RuntimeError).  fsp_last_error() returns thread-local text.
 *   - bf16 tensors, fp32 softmax statistics; row strides are in ELEMENTS.
 */
#ifndef FLEXSP_B200_H_
#define FLEXSP_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSP_OK 0
#define FSP_ERR_INVALID (-1)
#define FSP_ERR_CUDA (-2)
#define FSP_ERR_UNSUPPORTED (-3)

#define FSP_ABI_VERSION 6

/* FspAttnFwd / FspAttnBwd .flags */
#define FSP_ATTN_NONCAUSAL 1

int fsp_abi_version(void);
const char* fsp_last_error(void);

/* ------------------------------------------------------------------ pack */
/* Row gather:  dst[i, :row_bytes] = src[index[i], :row_bytes]; index[i] < 0 -> zero row.
 * Packs loader-order rows into the group-packed, rank-sharded layout.
 * Strides in bytes; row_bytes, strides and base pointers must be multiples of 16. */
int fsp_pack_rows(const void* src, int64_t src_stride_bytes, void* dst, int64_t dst_stride_bytes,
                  const int32_t* d_index, int64_t n_rows, int64_t row_bytes, void* stream);
/* Row scatter (inverse):  dst[index[i], :] = src[i, :] for index[i] >= 0. */
int fsp_unpack_rows(const void* src, int64_t src_stride_bytes, void* dst, int64_t dst_stride_bytes,
                    const int32_t* d_index, int64_t n_rows, int64_t row_bytes, void* stream);

/* Per-plan data scatter (ABI 5; "scatters the data into the corresponding
 * group"): the data loader shards a step's sequences over the ranks before the plan is
 * known (layout.loader_shards: round-robin); each micro-batch's rows must then reach the
 * members of the groups that own them.  d_routes is int32 [n_routes][3] =
 * {src_row, dst_rank, dst_row}: row src_row of the local shard (row stride
 * src_stride_bytes) is stored at row dst_row of peer_dst[dst_rank] (that rank's input
 * buffer mapped into this process; the own rank's entry is its local buffer).  The caller
 * brackets the scatter with fsp_group_barrier over all ranks (destination free / data
 * landed).  Strides, row_bytes and pointers: multiples of 16. */
int fsp_scatter_rows(const void* src, int64_t src_stride_bytes, void* const* peer_dst,
                     int32_t n_peers, int64_t dst_stride_bytes, const int32_t* d_routes,
                     int64_t n_routes, int64_t row_bytes, void* stream);

/* ------------------------------------------------------------------ all-to-all */
/* One Ulysses exchange inside an SP group of `degree` ranks on one NVSwitch domain.
 *
 * seq2head (Eq. 2): rank r holds rows [r*R, (r+1)*R) of the group-packed sequence with
 *   all H heads ([R, n_mats, H, D] at src, row stride src_stride elements); after the
 *   exchange rank j holds all degree*R rows for heads [j*H/d, (j+1)*H/d) in
 *   [degree*R, n_mats, H/d, D] at its recv buffer.  `peer_dst[j]` is rank j's recv buffer
 *   mapped into this process (symmetric memory); the local rank's own slice is copied
 *   locally.  If `d_src_index` is non-null the pack is fused: local row i is read from
 *   src row d_src_index[i] (negative -> zero pad row).
 * head2seq (Eq. 4): the inverse.  Rank r holds all degree*R rows for its heads
 *   ([degree*R, n_mats, H/d, D] at src); for every rank j it writes rows [j*R, (j+1)*R)
 *   into peer_dst[j] ([R, n_mats, H, D]) at head offset r*H/d.  If `d_dst_index` is
 *   non-null the unpack is fused: d_dst_index is [degree][R] — the unpack tables of all
 *   group members — and shard row i of member j lands in its destination row
 *   d_dst_index[j*R + i] (negative -> dropped, i.e. a pad row).
 *
 * Uneven heads (ABI 3): when head_begin[degree] != 0, member j owns heads
 *   [head_begin[j], head_begin[j+1]) (e.g. 52 heads at d=8: 7,7,7,7,6,6,6,6 — the 30B
 *   shape) instead of [j*H/d, (j+1)*H/d).  The head-sharded side then
 *   spaces its n_mats matrices hmax*D elements apart, hmax = max_j of the head counts
 *   (member j uses the first H_j heads of each); all zero = the even split.
 */
typedef struct FspA2A {
  int32_t degree;        /* d, power of two, 1..8 */
  int32_t rank;          /* rank inside the group, 0..d-1 */
  int32_t rows_per_rank; /* R = T_g / d (T_g padded to a multiple of d) */
  int32_t n_mats;        /* 3 for q,k,v; 1 for o / do */
  int32_t n_heads;       /* H (total; divisible by d unless head_begin is set) */
  int32_t head_dim;      /* D */
  int64_t src_stride;    /* elements between consecutive source rows */
  int64_t dst_stride;    /* elements between consecutive destination rows */
  int32_t head_begin[9]; /* optional uneven split: prefix offsets, [0..degree]; zeros = even */
} FspA2A;

int fsp_a2a_seq2head(const FspA2A* a, const void* src, void* const* peer_dst,
                     const int32_t* d_src_index, void* stream);
int fsp_a2a_head2seq(const FspA2A* a, const void* src, void* const* peer_dst,
                     const int32_t* d_dst_index, void* stream);
/* Group barrier over peer-mapped signal words: member `rank` of `degree` publishes
 * `epoch` to every member's slot [slot_base + rank] (system-scope release) and waits
 * until its own slots [slot_base, slot_base + degree) all reach `epoch` (acquire;
 * wrap-safe >=).  peer_signal[j] is member j's signal array mapped into this process;
 * a group occupying global ranks [r0, r0+d) uses slot_base = r0, so every rank owns one
 * slot per peer regardless of how the plan regroups ranks. */
int fsp_group_barrier(uint32_t* const* peer_signal, int32_t degree, int32_t rank,
                      int32_t slot_base, uint32_t epoch, void* stream);

/* ------------------------------------------------------------------ attention */
/* Fused head->seq exchange (Eq. 4) in an attention epilogue (ABI 4).
 * When degree > 0 the kernel stores every output row t of the group-packed sequence (its
 * own row index, 0 <= t < degree*rows_per_rank) for its heads ALSO into group member
 * r = t / rows_per_rank's sequence-sharded buffer peer_dst[r] (mapped into this process,
 * rows of n_mats matrices: matrix m of destination row u starts at element
 * u*dst_stride + m*mat_stride) at row d_unpack[t] (< 0: pad row, dropped) and heads
 * [head_offset, head_offset + n_heads).  d_unpack is the group's unpack table
 * ([degree][rows_per_rank], the one fsp_a2a_head2seq takes), so one fused launch does
 * what the attention launch followed by fsp_a2a_head2seq does, with the NVLink stores
 * issued tile by tile while other tiles still compute.  The caller still closes the
 * exchange with fsp_group_barrier.  Forward: O is matrix 0 (o is still written locally,
 * the backward needs it).  Backward: dQ, dK, dV are matrices 0, 1, 2 and the local
 * dq / dk / dv pointers may be NULL. */
typedef struct FspHeadScatter {
  int32_t degree;          /* 0 = off; else 1..8 */
  int32_t rows_per_rank;   /* R */
  int32_t head_offset;     /* first head of this member in the destination rows */
  int32_t reserved;
  int64_t dst_stride;      /* elements between destination rows */
  int64_t mat_stride;      /* elements between the matrices of one destination row */
  const int32_t* d_unpack; /* device [degree * rows_per_rank] */
  void* peer_dst[8];       /* member r's destination base, peer-mapped */
} FspHeadScatter;

/* Varlen causal attention over cu_seqlens-packed sequences (flash-attn varlen
 * semantics: causal inside each sequence, no cross-sequence attention, scale
 * default 1/sqrt(head_dim)).  head_dim must be 64 or 128.
 * Layouts: q/k/v/o/do/dq/dk/dv rows are tokens, each row holds n_heads*head_dim
 * contiguous bf16 values; consecutive rows are `*_stride` elements apart (so a
 * packed [T, 3, H, D] qkv buffer is addressed with q = base, k = base + H*D,
 * v = base + 2*H*D, stride 3*H*D).  lse is fp32 [n_heads, total_rows] (log-sum-exp
 * in natural-log units).  Tiles: 128 query rows; `d_tiles` is the schedule built by
 * fsp_attn_schedule() and uploaded by the caller. */
typedef struct FspAttnFwd {
  const void* q;
  const void* k;
  const void* v;
  void* o;
  float* lse;
  int64_t q_stride, k_stride, v_stride, o_stride;
  const int32_t* d_cu_seqlens; /* [n_seq+1], int32, device: lengths as prefix sums */
  const int32_t* d_seq_starts; /* optional [n_seq] first row of each sequence (NULL: the
                                  cu_seqlens offsets), so sequences can be read in place
                                  from any row order that keeps each one contiguous */
  const int32_t* d_tiles;      /* schedule from fsp_attn_schedule, device */
  int32_t n_tiles;
  int32_t n_seq;
  int32_t total_rows;
  int32_t n_heads;
  int32_t head_dim;
  float softmax_scale;
  FspHeadScatter scatter; /* ABI 4: optional fused head->seq of O (degree 0 = off) */
  int32_t flags;          /* ABI 6: FSP_ATTN_NONCAUSAL = every query row of a sequence sees
                             every key row of it (a context-parallel block whose keys all
                             precede its queries); 0 = causal */
} FspAttnFwd;

typedef struct FspAttnBwd {
  const void* q;
  const void* k;
  const void* v;
  const void* o;
  const void* dout;
  const float* lse;
  void* dq;
  void* dk;
  void* dv;
  int64_t q_stride, k_stride, v_stride, o_stride, do_stride, dq_stride, dk_stride, dv_stride;
  float* dq_accum;    /* workspace fp32 [n_heads, total_rows, head_dim] */
  float* delta;       /* workspace fp32 [n_heads, total_rows] */
  const int32_t* d_cu_seqlens;
  const int32_t* d_seq_starts; /* optional, as in FspAttnFwd */
  const int32_t* d_tiles; /* kv-tile schedule (same format as forward) */
  int32_t n_tiles;
  int32_t n_seq;
  int32_t total_rows;
  int32_t n_heads;
  int32_t head_dim;
  float softmax_scale;
  FspHeadScatter scatter; /* ABI 4: optional fused head->seq of dQ/dK/dV (degree 0 = off) */
  int32_t flags;          /* ABI 6: FSP_ATTN_NONCAUSAL (as in FspAttnFwd) */
} FspAttnBwd;

/* CTA schedule: writes n entries of two int32 {seq << 16 | unit, head} to tiles_host
 * (2*capacity words; NULL to query) and returns n (negative on error).  kind
 * FSP_SCHED_FWD: units are query tiles (128 rows; 256-row tile pairs when head_dim is
 * 128, matching fsp_attn_fwd's kernel); FSP_SCHED_BWD: 128-row kv tiles.  Sequences
 * longest first; within a sequence one head at a time, heaviest unit first (causal cost:
 * forward unit t grows with t, backward kv tile t costs n_tiles - t), so the resident
 * CTAs share one head's operands in L2.  n_tiles in FspAttnFwd/FspAttnBwd is this n. */
#define FSP_SCHED_FWD 0
#define FSP_SCHED_BWD 1
int32_t fsp_attn_schedule(const int32_t* cu_seqlens_host, int32_t n_seq, int32_t n_heads,
                          int32_t head_dim, int32_t kind, int32_t* tiles_host, int32_t capacity);
int fsp_attn_fwd(const FspAttnFwd* a, void* stream);
int fsp_attn_bwd(const FspAttnBwd* a, void* stream);
/* Bytes of fp32 scratch one fsp_attn_bwd call needs from its caller: dq_accum
 * [n_heads, total_rows, head_dim] + delta [n_heads, total_rows] (the library never
 * allocates).  Negative sizes -> FSP_ERR_INVALID. */
int64_t fsp_attn_bwd_workspace_bytes(int32_t total_rows, int32_t n_heads, int32_t head_dim);

/* ------------------------------------------------------------------ layout check */
/* Host-side validation of one group member's pack index (or a member's slice of an unpack
 * table): every entry is -1 (pad row) or a loader-order local row in [0, n_local), and the
 * non-negative entries hit each local row exactly once.  Returns 0 or FSP_ERR_INVALID
 * (message in fsp_last_error).  The executor runs it on every table it uploads. */
int fsp_layout_check(const int32_t* index_host, int64_t n_entries, int64_t n_local);

/* ------------------------------------------------------------------ self-test */
/* Single 128x128xK UMMA tile through TMA+tcgen05, used by the tests to pin the
 * descriptor formats.  mode 0: A[128,K] B[128,K] (both K-major) C=A*B^T;
 * 1: A[128,K], B[K,128] (MN-major) C=A*B; 2: as 1 with A staged in TMEM;
 * 3: A[K,128] (MN-major), B[128,K] C=A^T*B^T. C is fp32 [128,128]. */
int fsp_selftest_umma(int32_t mode, const void* a, const void* b, float* c, int32_t k,
                      void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FLEXSP_B200_H_ */
