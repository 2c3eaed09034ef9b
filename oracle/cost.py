"""Table 2 communication-overhead closed forms (oracle; test infrastructure only).

PAPER.md:212 (§4.1.1) — n nodes of w GPUs, N = w*n; embedding of size M;
gradient density alpha; uniform bandwidth B and start latency beta.
Table 2, derivations at PAPER.md:215 (AllReduce), 217 (PS),
239 (AllGather), 241-243 (AlltoAll).
"""


def cost_allreduce(N, M, B, beta):
    """2(N-1)(M/(NB) + beta)."""
    return 2 * (N - 1) * (M / (N * B) + beta)


def cost_ps(N, S, alpha, M, B, beta):
    """2N(alpha M/(S B) + beta); lower bound at S = n."""
    return 2 * N * (alpha * M / (S * B) + beta)


def cost_allgather(N, alpha, M, B, beta):
    """(N-1)(alpha M / B + beta)."""
    return (N - 1) * (alpha * M / B + beta)


def cost_alltoall(N, alpha, M, B, beta):
    """two AlltoAlls, each N-1 exchanges of alpha M / N:
    2(N-1)(alpha M/(N B) + beta)."""
    return 2 * (N - 1) * (alpha * M / (N * B) + beta)


def alltoall_bandwidth_numerator(N, alphaM):
    """Elements one rank sends in ONE AlltoAll of total payload alphaM
    ('each exchange amount will be alpha M / N', N-1 exchanges)."""
    return (N - 1) * alphaM / N


def allgather_bandwidth_numerator(N, alphaM):
    """'summing up the transmitted data size to (N-1) alpha M'."""
    return (N - 1) * alphaM


def beta_threshold_allgather_vs_alltoall(N, alpha, M, B):
    """beta at which cost_allgather == cost_alltoall (AllGather
    wins only for small N and long beta).  Solve
    (N-1)(aM/B + b) = 2(N-1)(aM/(NB) + b)  ->  b = aM/B (1 - 2/N)."""
    return alpha * M / B * (1.0 - 2.0 / N)
