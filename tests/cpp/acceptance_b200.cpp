// The reference's acceptance gate (/root/reference/proj/tests/acceptance_main.cpp, all ten
// checks) compiled UNMODIFIED against the B200 drop-in: its hot-path calls (run_stream /
// StreamEngine, build_index, HierIndex, TieredStore, Maintainer, retrieve, oracle_flat_topk,
// retrieve_token_baseline, updated_stats, tau) resolve to include/kvclust_b200*.hpp and run on
// the GPU engine (libkvclust_b200.so over libkvc.so). The reference's non-hot-path modules it
// also calls (workload: gen_stream / save_trace, clustering: spherical_kmeans, harness: cmd_run,
// report) are the reference's own sources, compiled against the drop-in headers (Makefile).
// Test infrastructure: built by tests/cpp/Makefile where /root/reference exists; the binary travels
// to the GPU box and tests/test_acceptance_gpu.py runs it.
#include "acceptance_main.cpp"  // from /root/reference/proj/tests (-I), not copied
