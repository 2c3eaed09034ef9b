// dense_queue.cu — deterministic priority issue rule + NCCL AllReduce on a
// side stream (see dense_queue.h).
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstring>

#include "dense_queue.h"

namespace {

struct Req {
  int32_t prio;
  int64_t seq;
  void* buf;
  int64_t count;
  emb_dtype dt;
  cudaEvent_t ready;
};

bool before(const Req& a, const Req& b) { return a.prio != b.prio ? a.prio < b.prio : a.seq < b.seq; }

// Shared by the pure rule and the live queue: append one request and return
// the requests that must be issued now (window rule), in issue order.
template <typename Issue>
void rule_push(std::vector<Req>& pending, const Req& r, int window, Issue issue) {
  pending.push_back(r);
  while ((int)pending.size() >= window) {
    auto it = std::min_element(pending.begin(), pending.end(), before);
    Req x = *it;
    pending.erase(it);
    issue(x);
  }
}

template <typename Issue>
void rule_flush(std::vector<Req>& pending, Issue issue) {
  std::sort(pending.begin(), pending.end(), before);
  for (const Req& x : pending) issue(x);
  pending.clear();
}

}  // namespace

void issue_rule_order(const int32_t* priorities, int32_t n, int32_t window, std::vector<int64_t>* order) {
  std::vector<Req> pending;
  order->clear();
  auto issue = [&](const Req& x) { order->push_back(x.seq); };
  for (int32_t i = 0; i < n; ++i) {
    Req r{priorities[i], i, nullptr, 0, EMB_FP32, nullptr};
    rule_push(pending, r, window, issue);
  }
  rule_flush(pending, issue);
}

// Completion events live in a ring of RING slots (ticket t -> slot t % RING),
// recycled as tickets advance, so a long run holds a fixed number of events
// and bytes; the issue log keeps the first LOG_CAP entries.
static constexpr int64_t RING = 1024;
static constexpr size_t LOG_CAP = 1 << 16;

struct DenseQueue {
  ncclComm_t comm = nullptr;
  cudaStream_t stream = nullptr;
  int window = 1;
  int64_t next_seq = 0;
  std::vector<Req> pending;
  cudaEvent_t done[RING] = {};      // slot of ticket t: t % RING
  int64_t slot_ticket[RING];        // ticket currently owning the slot (-1: none)
  bool slot_issued[RING] = {};
  std::vector<int64_t> log;
  emb_status err = EMB_OK;
};

DenseQueue* dense_queue_create(const uint8_t* nccl_id, int world, int rank, int window) {
  DenseQueue* q = new DenseQueue();
  q->window = window < 1 ? 1 : window;
  ncclUniqueId id;
  memcpy(&id, nccl_id, sizeof(id));
  if (ncclCommInitRank(&q->comm, world, id, rank) != ncclSuccess) {
    fprintf(stderr, "[embrace] ncclCommInitRank failed\n");
    delete q;
    return nullptr;
  }
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  bool ok = cudaStreamCreateWithPriority(&q->stream, cudaStreamNonBlocking, hi) == cudaSuccess;
  for (int64_t i = 0; i < RING; ++i) {
    q->slot_ticket[i] = -1;
    if (ok) ok = cudaEventCreateWithFlags(&q->done[i], cudaEventDisableTiming) == cudaSuccess;
  }
  if (!ok) {
    dense_queue_destroy(q);
    return nullptr;
  }
  return q;
}

static void do_issue(DenseQueue* q, const Req& x) {
  if (q->err != EMB_OK) return;
  if (x.ready && cudaStreamWaitEvent(q->stream, x.ready, 0) != cudaSuccess) { q->err = EMB_ERR_CUDA; return; }
  ncclDataType_t t = x.dt == EMB_BF16 ? ncclBfloat16 : ncclFloat32;
  if (ncclAllReduce(x.buf, x.buf, (size_t)x.count, t, ncclAvg, q->comm, q->stream) != ncclSuccess) {
    q->err = EMB_ERR_NCCL;
    return;
  }
  if (cudaEventRecord(q->done[x.seq % RING], q->stream) != cudaSuccess) { q->err = EMB_ERR_CUDA; return; }
  q->slot_issued[x.seq % RING] = true;
  if (q->log.size() < LOG_CAP) q->log.push_back(x.seq);
}

emb_status dense_queue_enqueue(DenseQueue* q, void* buf, int64_t count, emb_dtype dt, int32_t prio,
                               cudaEvent_t ready, int64_t* ticket) {
  if (q->err != EMB_OK) return q->err;
  const int64_t slot = q->next_seq % RING;
  // the slot's previous ticket (next_seq - RING) must have been issued
  if (q->slot_ticket[slot] >= 0 && !q->slot_issued[slot]) return EMB_ERR_CAPACITY;
  Req r{prio, q->next_seq++, buf, count, dt, ready};
  q->slot_ticket[slot] = r.seq;
  q->slot_issued[slot] = false;
  *ticket = r.seq;
  rule_push(q->pending, r, q->window, [&](const Req& x) { do_issue(q, x); });
  return q->err;
}

emb_status dense_queue_flush_all(DenseQueue* q) {
  rule_flush(q->pending, [&](const Req& x) { do_issue(q, x); });
  return q->err;
}

emb_status dense_queue_wait(DenseQueue* q, int64_t ticket, cudaStream_t consumer) {
  if (q->err != EMB_OK) return q->err;
  if (ticket < 0 || ticket >= q->next_seq) return EMB_ERR_INVALID_ARG;
  const int64_t slot = ticket % RING;
  if (q->slot_ticket[slot] != ticket) return EMB_ERR_STATE;  // expired: RING newer tickets since
  if (!q->slot_issued[slot]) return EMB_ERR_STATE;          // still pending: flush first
  return cudaStreamWaitEvent(consumer, q->done[slot], 0) == cudaSuccess ? EMB_OK : EMB_ERR_CUDA;
}

emb_status dense_queue_wait_all(DenseQueue* q, cudaStream_t consumer) {
  if (q->err != EMB_OK) return q->err;
  cudaEvent_t ev;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return EMB_ERR_CUDA;
  emb_status st = EMB_OK;
  if (cudaEventRecord(ev, q->stream) != cudaSuccess || cudaStreamWaitEvent(consumer, ev, 0) != cudaSuccess)
    st = EMB_ERR_CUDA;
  cudaEventDestroy(ev);
  return st;
}

void dense_queue_issue_log(DenseQueue* q, std::vector<int64_t>* log) { *log = q->log; }

void dense_queue_destroy(DenseQueue* q) {
  if (!q) return;
  if (q->stream) cudaStreamSynchronize(q->stream);
  for (cudaEvent_t e : q->done)
    if (e) cudaEventDestroy(e);
  if (q->comm) ncclCommDestroy(q->comm);
  if (q->stream) cudaStreamDestroy(q->stream);
  delete q;
}
