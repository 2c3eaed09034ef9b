// dense_queue.h — Horizontal Scheduling's priority queue for dense gradients
// ("we change the FIFO queue to a priority
// queue [...] The dense blocks get priority according to the FP dependency
// order", "we hold a priority queue and a communication thread").
//
// The paper's communication thread pops whatever is ready, which depends on
// timing and could issue collectives in a different order on each rank.  Here
// the issue order is a pure function of the enqueue sequence (reading R16):
// after each enqueue, while >= W requests are pending, the smallest
// (priority, seq) is issued; flush issues the rest in that order.  Issuing =
// the comm stream waits for the block's ready event, then ncclAllReduce(avg).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/embrace.h"

struct DenseQueue;

// Pure rule: the order (seq numbers) in which requests with these priorities,
// enqueued in array order, are issued under window W (then flushed).
void issue_rule_order(const int32_t* priorities, int32_t n, int32_t window, std::vector<int64_t>* order);

DenseQueue* dense_queue_create(const uint8_t* nccl_id, int world, int rank, int window);
emb_status dense_queue_enqueue(DenseQueue* q, void* buf, int64_t count, emb_dtype dt, int32_t prio,
                               cudaEvent_t ready, int64_t* ticket);
emb_status dense_queue_flush_all(DenseQueue* q);
emb_status dense_queue_wait(DenseQueue* q, int64_t ticket, cudaStream_t consumer);
emb_status dense_queue_wait_all(DenseQueue* q, cudaStream_t consumer);
void dense_queue_issue_log(DenseQueue* q, std::vector<int64_t>* log);
void dense_queue_destroy(DenseQueue* q);
