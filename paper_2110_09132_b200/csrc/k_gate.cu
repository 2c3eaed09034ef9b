// k_gate.cu — the peer-flag gates of the N > 1 exchange (DESIGN.md "Flag
// protocol", "Liveness").
//
// Every cross-GPU wait of the path happens in a gate: ONE CTA of one warp,
// launched on the stream right before the kernel that consumes the peers'
// data.  The gate (a) starts after its stream predecessor completed
// (griddepcontrol.wait), so that producer's stores are performed, and
// publishes the producer's flag to every peer; (b) spins until every peer's
// matching flag arrived; (c) only then lets its dependent launch
// (griddepcontrol.launch_dependents after the wait).  The compute kernels
// themselves never spin.
//
// Why a separate kernel: a wide kernel whose CTAs spin occupies SMs while it
// waits, and two such kernels on different streams of two GPUs can starve the
// very kernels their peers wait for (observed: a side-stream merge spinning on
// every SM of one GPU while the other GPU's forward spun on every SM — a
// cross-GPU deadlock, EMB_ERR_TIMEOUT).  Gates hold one warp while waiting, so
// every other kernel can always be scheduled and every wait eventually
// resolves.  The only other spinning kernel is mark (N <= 8 CTAs).
#include <stddef.h>

#include "kernels.cuh"

namespace emb {

__global__ void __launch_bounds__(32) gate_kernel(DevCtx c, int p, int kind, int flag_arg) {
  EMB_TR_ENTRY();
  pdl_wait();
  if (threadIdx.x == 0) {
    switch (kind) {
      case GATE_FWD: {
        // forward(t): every owner (this rank included) must have applied the
        // prior part of t-1 (published by the last CTA of its merge(part 0),
        // k_bwd.cu) and the scheduled part of t-2 (SPLIT: GATE_DEFDONE on its
        // side stream; otherwise with prior_done)
        const uint32_t t = c.t_rec[p ^ 1] + 1;
        EMB_TR_BEGIN(10 + kind, t);
        EMB_TR_WAITED(10 + kind, t);  // past griddepcontrol.wait (predecessor complete)
        Flags* f = flags_of(c, c.r);
        wait_all(c, f->prior_done, t - 1, 1);
        wait_all(c, f->def_done, t - 2, 2);
        if (flag_arg & 1) wait_local(c, c.marked + (p ^ 1), t - 1, 3);  // the prefetch copy this forward checks
        if (flag_arg & 2) c.fwd_dd[p] = ((int)(ld_acquire_gpu(c.sorted + p) - t) >= 0) ? 1u : 0u;  // dedup iff sorted
        EMB_TR_END(10 + kind, t);
        break;
      }
      case GATE_SORT: {
        // ids of batch tt (parity p).  flag_arg bits: 1 = the predecessor (the
        // forward or markpush) pushed this rank's ids: publish them; 2 = wait
        // for every source's ids; 4 (SPLIT) = the routing tables of parity p are
        // free once this rank's scheduled push of tt-2 (side stream) is past.
        // 16 = launched from a backward (batch t+1): one past the sort of t on
        // this stream; else from a forward (batch t), after it
        const uint32_t tt = (flag_arg & 16) ? __ldcg(c.sorted + (p ^ 1)) + 1 : c.t_rec[p ^ 1] + 1;
        EMB_TR_BEGIN(10 + kind, tt);
        EMB_TR_WAITED(10 + kind, tt);
        if (flag_arg & 1) publish(c, EMB_FLAG_OFF(ids), tt);
        if (flag_arg & 2) wait_all(c, flags_of(c, c.r)->ids, tt, 4);
        // (the scheduled merge reads the merge plan, not the routing tables, so
        // only this rank's scheduled push of tt-2 must be past them)
        if ((flag_arg & 4) && c.mode == SPLIT && tt >= 3) wait_local(c, c.seq + SEQ_DEFPUSHED, tt - 2, 5 * 16);
        // 8 (SPLIT): the merge plan / D_next tags of parity tt-1 are free once
        // this rank's scheduled merge of tt-3 is done (the work may start before
        // the forward of tt-1 when emb_prefetch forked it early)
        if ((flag_arg & 8) && c.mode == SPLIT && tt >= 4)
          wait_flag(c, &flags_of(c, c.r)->def_done[c.r], tt - 3, 5 * 16 + 1);
        EMB_TR_END(10 + kind, tt);
        break;
      }
      case GATE_PUB0:
      case GATE_PUB1: {
        // owner merge of part (prior / scheduled): the sender pass preceding this
        // gate completed; every sender's pass must have completed
        const uint32_t t = c.t_rec[p];
        EMB_TR_BEGIN(10 + kind, t);
        EMB_TR_WAITED(10 + kind, t);  // past griddepcontrol.wait (predecessor complete)
        const int part = (kind == GATE_PUB1) ? 1 : 0;
        if (!part) st_release_gpu(c.seq + SEQ_APPLIED, t);     // the apply of t completed (side stream waits)
        else st_release_gpu(c.seq + SEQ_DEFPUSHED, t);          // defpush(t) no longer needs the routing tables
        publish(c, part ? EMB_FLAG_OFF(pub[1]) : EMB_FLAG_OFF(pub[0]), t);
        wait_all(c, flags_of(c, c.r)->pub[part], t, 6 + part);
        if (!part) wait_local(c, c.marked + p, t, 8 * 16 + 2);  // the merge plan of t (aux stream) is complete
        EMB_TR_END(10 + kind, t);
        break;
      }
      case GATE_MARKED: {
        // apply of t (SPLIT): the D_next tags of t+1 are complete (mark, aux stream)
        const uint32_t t = c.t_rec[p];
        EMB_TR_BEGIN(10 + kind, t);
        EMB_TR_WAITED(10 + kind, t);  // past griddepcontrol.wait (predecessor complete)
        wait_local(c, c.marked + p, t, 8 * 16);
        EMB_TR_END(10 + kind, t);
        break;
      }
      case GATE_SORTED: {
        // coalesce of t: the sort of batch t (aux stream) completed — a local
        // flag instead of a host event keeps the main stream's PDL chain; at
        // N == 1 also the prefetch check (fingerprints of fwd(t) and sort(t))
        const uint32_t t = c.t_rec[p];
        EMB_TR_BEGIN(10 + kind, t);
        EMB_TR_WAITED(10 + kind, t);  // past griddepcontrol.wait (predecessor complete)
        wait_local(c, c.sort_count + p, (t + 1) / 2, 9 * 16);  // one sort of parity p per iteration
        unsigned* f = c.fp + p * 4;
        if (f[0] != f[2] || f[1] != f[3]) atomicOr(c.err, ERR_STATE);
        f[0] = f[1] = f[2] = f[3] = 0;
        // forward(t) and sort(t) done, next_ids of backward(t) ready in stream
        // order: the aux / side streams may start backward(t)'s work
        st_release_gpu(c.seq + SEQ_BWD, t);
        EMB_TR_END(10 + kind, t);
        break;
      }
      case GATE_DEFDONE: {
        // the scheduled merge of t (this stream's predecessor) completed
        const uint32_t t = c.t_rec[p];
        EMB_TR_BEGIN(10 + kind, t);
        EMB_TR_WAITED(10 + kind, t);  // past griddepcontrol.wait (predecessor complete)
        publish(c, EMB_FLAG_OFF(def_done), t);
        EMB_TR_END(10 + kind, t);
        break;
      }
      default:
        atomicOr(c.err, ERR_STATE);
    }
  }
  __syncwarp();
  pdl_trigger();  // after the wait: the dependent's CTAs must not launch (and sit) earlier
}

cudaError_t launch_gate(const DevCtx& c, int p, int kind, int flag_arg, cudaStream_t s) {
  return launch_pdl(gate_kernel, dim3(1), dim3(32), 0, s, c, p, kind, flag_arg);
}

cudaError_t preload_gate() { return preload((const void*)gate_kernel); }

}  // namespace emb
