// concurrency_table.cpp -- the paper's concurrency experiment ("Raw FA classifier latency
// (median ms, no compression)", C = 1 / 10 / 20 concurrent requests at 512 .. 32K tokens) on one B200, driven
// through the model-backed ClassifierSet (include/routefast_b200/classifiers.hpp) in StreamHandler's call order
// (reference proj/core/src/stream.cpp:438-443: jailbreak, PII, domain; no compression here, so all three see the
// full text).  The reference serves every request on its own thread with its own StreamHandler
// (service.cpp:141); its stub classifiers are stateless and shared.  A model session is not re-entrant, so each
// in-flight request owns one ClassifierSet (a session pool of size C); the three weight blobs are generated once
// and shared by the pool.  Random-init weights, synthetic text (one hashed word per token).
//
// usage: concurrency_table [max_tokens_list e.g. 512,2048,8192] [C list e.g. 1,10,20]
// prints one JSON line per (tokens, C): median / p90 latency of one classifier call and of the 3-call request.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "routefast_b200/classifiers.hpp"

namespace rf = routefast_b200;
using Clock = std::chrono::steady_clock;

static std::vector<int> parse_list(const char* s) {
    std::vector<int> v;
    std::stringstream ss(s);
    std::string tok;
    while (std::getline(ss, tok, ',')) v.push_back(std::atoi(tok.c_str()));
    return v;
}

static std::string make_text(int tokens, unsigned seed) {
    std::string t;
    t.reserve(static_cast<size_t>(tokens) * 7);
    unsigned x = seed * 2654435761u + 12345u;
    for (int i = 0; i < tokens; ++i) {
        x = x * 1664525u + 1013904223u;
        t += "w" + std::to_string(x % 50000u) + " ";
    }
    return t;
}

struct Barrier {
    std::mutex m;
    std::condition_variable cv;
    int count, waiting = 0, gen = 0;
    explicit Barrier(int n) : count(n) {}
    void wait() {
        std::unique_lock<std::mutex> lk(m);
        const int g = gen;
        if (++waiting == count) {
            waiting = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

static double pct(std::vector<double> v, double p) {
    std::sort(v.begin(), v.end());
    return v.empty() ? 0.0 : v[std::min(v.size() - 1, static_cast<size_t>(p * (v.size() - 1) + 0.5))];
}

int main(int argc, char** argv) {
    const std::vector<int> lens = parse_list(argc > 1 ? argv[1] : "512,2048,8192,16384,32768");
    const std::vector<int> concs = parse_list(argc > 2 ? argv[2] : "1,10,20");
    const int max_c = *std::max_element(concs.begin(), concs.end());
    rf_clf_config cfg;
    rf_clf_config_default(&cfg);
    cfg.vocab_size = 50368;
    const std::vector<std::string> domains = {"general", "code", "math", "medical", "legal"};

    // three models (safety, PII, domain: BASELINE config 3), one weight blob each, shared by the pool
    rf_clf_config cj = cfg, cp = cfg, cd = cfg;
    cj.n_labels = 2;
    cp.n_labels = 3;
    cd.n_labels = static_cast<int>(domains.size());
    const std::vector<float> wj = rf::random_init_weights(cj, 7), wp = rf::random_init_weights(cp, 8), wd = rf::random_init_weights(cd, 9);
    std::vector<rf::ClassifierSet> pool(static_cast<size_t>(max_c));
    for (auto& set : pool) {
        set.jailbreak = std::make_shared<const rf::ModelJailbreakClassifier>(std::make_shared<const rf::ModelSession>(cj, wj, 0), 0.5);
        set.pii = std::make_shared<const rf::ModelPiiClassifier>(std::make_shared<const rf::ModelSession>(cp, wp, 0));
        set.domain = std::make_shared<const rf::ModelDomainClassifier>(std::make_shared<const rf::ModelSession>(cd, wd, 0), domains);
    }
    std::fprintf(stderr, "pool of %d ClassifierSets ready\n", max_c);

    for (int tokens : lens) {
        for (int C : concs) {
            const int rounds = tokens >= 16384 ? 3 : 5;
            std::vector<std::vector<double>> call_ms(static_cast<size_t>(C)), req_ms(static_cast<size_t>(C));
            Barrier bar(C);
            std::atomic<int> errors{0};
            std::vector<std::thread> th;
            for (int t = 0; t < C; ++t)
                th.emplace_back([&, t] {
                    const std::string text = make_text(tokens, static_cast<unsigned>(t + 1));
                    const rf::ClassifierSet& set = pool[static_cast<size_t>(t)];
                    try {
                        for (int w = 0; w < 2; ++w) {  // a shape is captured into a CUDA graph on its second call
                            set.jailbreak->classify(text);
                            set.pii->classify(text);
                            set.domain->classify(text);
                        }
                        bar.wait();
                        for (int r = 0; r < rounds; ++r) {
                            const auto t0 = Clock::now();
                            set.jailbreak->classify(text);
                            const auto t1 = Clock::now();
                            set.pii->classify(text);
                            set.domain->classify(text);
                            const auto t2 = Clock::now();
                            call_ms[static_cast<size_t>(t)].push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
                            req_ms[static_cast<size_t>(t)].push_back(std::chrono::duration<double, std::milli>(t2 - t0).count());
                        }
                    } catch (const std::exception& e) {
                        std::fprintf(stderr, "thread %d: %s\n", t, e.what());
                        ++errors;
                        bar.wait();
                    }
                });
            for (auto& x : th) x.join();
            std::vector<double> calls, reqs;
            for (int t = 0; t < C; ++t) {
                calls.insert(calls.end(), call_ms[static_cast<size_t>(t)].begin(), call_ms[static_cast<size_t>(t)].end());
                reqs.insert(reqs.end(), req_ms[static_cast<size_t>(t)].begin(), req_ms[static_cast<size_t>(t)].end());
            }
            std::printf("{\"tokens\": %d, \"C\": %d, \"classifier_call_ms_median\": %.2f, \"classifier_call_ms_p90\": %.2f, "
                        "\"request_3_classifiers_ms_median\": %.2f, \"request_3_classifiers_ms_p90\": %.2f, \"samples\": %zu, \"errors\": %d}\n",
                        tokens, C, pct(calls, 0.5), pct(calls, 0.9), pct(reqs, 0.5), pct(reqs, 0.9), calls.size(), errors.load());
            std::fflush(stdout);
        }
    }
    return 0;
}
