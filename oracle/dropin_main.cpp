// TEST INFRASTRUCTURE: the link-substitution proof of the drop-in.
//
// One driver, linked twice by oracle/Makefile:
//   _ref/pipeline_ref  = this main + ALL reference objects (the pure reference)
//   _ref/pipeline_b200 = this main + the reference objects minus engine.o/cluster.o
//                        + paper_2512_00398_b200/dropin (engine_b200.o, cluster_b200.o)
//                        + libpgb200.so
// Both run the reference's own create_task + execute_task (src/pipeline.cpp:32-119)
// on the same SIGPROC file and write the reference's .cand text; the test compares
// the files byte for byte.
//
// usage: pipeline_* in.fil out.cand dm_lo dm_hi dm_step boxcar_max baseline_s nsamps_chunk n_workers [rfi]
// PG_TIMING_OUT=path: EngineConfig::timing_sink appends one line per TrialTiming record
// ("trial dedisperse baseline normalize boxcar peaks", ms) to path.
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>

#include "pulsegrid/pipeline.hpp"

int main(int argc, char** argv) {
    using namespace pulsegrid;
    if (argc != 10 && argc != 11) {
        std::fprintf(stderr, "usage: %s in.fil out.cand dm_lo dm_hi dm_step boxcar baseline_s chunk workers\n",
                     argv[0]);
        return 2;
    }
    try {
        SearchParams p;
        p.dm_lo = std::atof(argv[3]);
        p.dm_hi = std::atof(argv[4]);
        p.spacing = LinearSpacing{std::atof(argv[5])};
        p.engine.boxcar_max = std::strtoull(argv[6], nullptr, 10);
        p.baseline_len_s = std::atof(argv[7]);
        p.nsamps_chunk = std::strtoull(argv[8], nullptr, 10);
        p.engine.n_workers = (std::uint32_t)std::atoi(argv[9]);
        p.engine.max_in_flight = p.engine.n_workers;  // parity mode (block size 1)
        const bool rfi = argc == 11 && std::atoi(argv[10]) != 0;  // reference defaults when on
        p.rfi_narrowband = rfi;
        p.rfi_broadband = rfi;
        std::FILE* tf = nullptr;
        std::mutex tf_mu;
        if (const char* tp = std::getenv("PG_TIMING_OUT")) {
            tf = std::fopen(tp, "w");
            if (!tf) throw std::runtime_error("cannot open PG_TIMING_OUT");
            p.engine.timing_sink = [&](const TrialTiming& t) {
                std::lock_guard<std::mutex> lk(tf_mu);
                std::fprintf(tf, "%zu %.6f %.6f %.6f %.6f %.6f\n", t.trial, t.dedisperse_ms, t.baseline_ms,
                             t.normalize_ms, t.boxcar_ms, t.peaks_ms);
            };
        }
        auto task = create_task(argv[1], p, argv[2]);
        BufferPool pool(p.engine.memory_budget);
        auto out = execute_task(task, pool);
        std::printf("{\"clusters\": %zu, \"chunks\": %zu, \"wall_ms\": %.3f, \"read_ms\": %.3f, "
                    "\"dm_loop_ms\": %.3f, \"cluster_ms\": %.3f, \"skipped\": %zu}\n",
                    out.candidates, task.chunks.size(), out.wall_ms, out.read_ms, out.dm_loop_ms,
                    out.cluster_ms, out.skipped_trials.size());
        if (tf) std::fclose(tf);
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
