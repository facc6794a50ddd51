// routefast_b200/classifiers.hpp -- model-backed implementation of the reference's pluggable classifier
// interface (reference: proj/core/include/routefast/classifiers.hpp:13-80), on the B200 through the native
// classifier session of librf_fa.so (include/rf_clf.h).  Header-only; link with -lrf_fa.
//
// Same names and fields as the reference: JailbreakSignal / PiiSignal / DomainSignal, the abstract
// JailbreakClassifier / PiiClassifier / DomainClassifier with `classify(std::string_view) const`, and
// ClassifierSet{jailbreak, pii, domain}.  Where the reference ships keyword stubs
// (StubJailbreakClassifier ..., classifiers.cpp:63-225) "so the whole routing pipeline is testable without
// a model runtime", this header supplies the model runtime behind the same interface; StreamHandler's call
// site (stream.cpp:438-443) is unchanged: jailbreak and PII see the full text, domain the compressed view.
//
// What is NOT the reference's: the tokenizer (none exists there; a deterministic word-hash tokenizer stands
// in) and the encoder weights (the reference has no model; random-init from a seed unless a weight blob is
// supplied).  With random weights the signals are arbitrary but deterministic -- the plumbing, the shapes,
// the error behaviour and the cost are what this layer pins down.
// There is no CPU fallback: a missing GPU surfaces as std::runtime_error at construction.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <memory>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "../rf_clf.h"

namespace routefast_b200 {

struct JailbreakSignal {  // classifiers.hpp:13-17
    bool flagged = false;
    double score = 0.0;
    std::string matched;
};
struct PiiSignal {  // classifiers.hpp:19-22
    bool flagged = false;
    std::vector<std::string> kinds;  // "ssn", "email", "credit_card"
};
struct DomainSignal {  // classifiers.hpp:24-27
    std::string label = "general";
    double score = 0.0;
};

class JailbreakClassifier {  // classifiers.hpp:32-36
public:
    virtual ~JailbreakClassifier() = default;
    virtual JailbreakSignal classify(std::string_view text) const = 0;
};
class PiiClassifier {  // classifiers.hpp:38-42
public:
    virtual ~PiiClassifier() = default;
    virtual PiiSignal classify(std::string_view text) const = 0;
};
class DomainClassifier {  // classifiers.hpp:44-48
public:
    virtual ~DomainClassifier() = default;
    virtual DomainSignal classify(std::string_view text) const = 0;
};

// Deterministic stand-in tokenizer: id 0 = [CLS], then one id per word (runs of alphanumerics) or
// punctuation byte, FNV-1a hashed into [1, vocab).  At most max_tokens ids (the tail is dropped).
inline std::vector<int64_t> hash_tokenize(std::string_view text, int32_t vocab, std::size_t max_tokens) {
    std::vector<int64_t> ids;
    ids.push_back(0);
    auto emit = [&](std::string_view w) {
        uint64_t h = 1469598103934665603ull;
        for (unsigned char ch : w) {
            h ^= static_cast<uint64_t>(std::tolower(ch));
            h *= 1099511628211ull;
        }
        ids.push_back(1 + static_cast<int64_t>(h % static_cast<uint64_t>(vocab - 1)));
    };
    std::size_t i = 0;
    while (i < text.size() && ids.size() < max_tokens) {
        const unsigned char ch = static_cast<unsigned char>(text[i]);
        if (std::isspace(ch)) {
            ++i;
        } else if (std::isalnum(ch) || ch >= 0x80) {
            std::size_t j = i;
            while (j < text.size() && (std::isalnum(static_cast<unsigned char>(text[j])) || static_cast<unsigned char>(text[j]) >= 0x80)) ++j;
            emit(text.substr(i, j - i));
            i = j;
        } else {
            emit(text.substr(i, 1));
            ++i;
        }
    }
    return ids;
}

// Random-init weight blob in rf_clf_create's tensor order (std 0.02, cls_w 0.05, norms 1, bias 0), the
// distribution classifier.py's init_weights uses (not the same random stream).
inline std::vector<float> random_init_weights(const rf_clf_config& c, uint64_t seed) {
    std::vector<float> w(rf_clf_weight_elems(&c));
    std::mt19937_64 rng(seed);
    std::normal_distribution<float> n02(0.0f, 0.02f), n05(0.0f, 0.05f);
    std::size_t o = 0;
    auto mat = [&](std::size_t n, std::normal_distribution<float>& dist) { for (std::size_t i = 0; i < n; ++i) w[o++] = dist(rng); };
    auto fill = [&](std::size_t n, float v) { for (std::size_t i = 0; i < n; ++i) w[o++] = v; };
    const std::size_t hid = c.hidden, mlp = c.mlp;
    mat(static_cast<std::size_t>(c.vocab_size) * hid, n02);  // tok_emb
    fill(hid, 1.0f);                                         // emb_norm
    fill(hid, 1.0f);                                         // final_norm
    mat(hid * hid, n02);                                     // head_dense
    fill(hid, 1.0f);                                         // head_norm
    mat(static_cast<std::size_t>(c.n_labels) * hid, n05);    // cls_w
    fill(c.n_labels, 0.0f);                                  // cls_b
    for (int l = 0; l < c.n_layers; ++l) {
        fill(hid, 1.0f);
        mat(3 * hid * hid, n02);
        mat(hid * hid, n02);
        fill(hid, 1.0f);
        mat(2 * mlp * hid, n02);
        mat(hid * mlp, n02);
    }
    return w;
}

// One classifier model on one GPU: RAII over rf_clf.  classify-style calls are serialised (the session is
// not re-entrant); the interface's `const` is kept by making the session state mutable.
class ModelSession {
public:
    ModelSession(const rf_clf_config& cfg, const std::vector<float>& weights, int device = 0, std::size_t max_tokens = 32768)
        : cfg_(cfg), max_tokens_(max_tokens) {
        if (rf_clf_create(&cfg_, weights.data(), weights.size(), device, &clf_) != RF_OK) throw std::runtime_error(rf_last_error());
    }
    ModelSession(const ModelSession&) = delete;
    ModelSession& operator=(const ModelSession&) = delete;
    ~ModelSession() { rf_clf_destroy(clf_); }

    // logits of one text
    std::vector<float> logits(std::string_view text) const {
        const std::vector<int64_t> ids = hash_tokenize(text, cfg_.vocab_size, max_tokens_);
        std::vector<float> out(static_cast<std::size_t>(cfg_.n_labels));
        std::lock_guard<std::mutex> lock(mu_);
        if (rf_clf_forward(clf_, ids.data(), nullptr, 1, static_cast<int64_t>(ids.size()), out.data()) != RF_OK)
            throw std::runtime_error(rf_last_error());
        last_tokens_ = ids.size();
        return out;
    }
    // a batch of texts, tail-padded to the longest with the attention mask the rewriter's pad-bias chain consumes
    std::vector<std::vector<float>> logits_batch(const std::vector<std::string_view>& texts) const {
        std::vector<std::vector<int64_t>> toks;
        std::size_t S = 1;
        for (auto t : texts) {
            toks.push_back(hash_tokenize(t, cfg_.vocab_size, max_tokens_));
            S = std::max(S, toks.back().size());
        }
        const std::size_t B = texts.size();
        std::vector<int64_t> ids(B * S, 0);
        std::vector<float> mask(B * S, 0.0f), flat(B * static_cast<std::size_t>(cfg_.n_labels));
        for (std::size_t b = 0; b < B; ++b)
            for (std::size_t i = 0; i < toks[b].size(); ++i) {
                ids[b * S + i] = toks[b][i];
                mask[b * S + i] = 1.0f;
            }
        std::lock_guard<std::mutex> lock(mu_);
        if (B > 0 && rf_clf_forward(clf_, ids.data(), mask.data(), static_cast<int64_t>(B), static_cast<int64_t>(S), flat.data()) != RF_OK)
            throw std::runtime_error(rf_last_error());
        std::vector<std::vector<float>> out(B);
        for (std::size_t b = 0; b < B; ++b) out[b].assign(flat.begin() + b * cfg_.n_labels, flat.begin() + (b + 1) * cfg_.n_labels);
        return out;
    }
    float last_forward_ms() const { return rf_clf_last_forward_ms(clf_); }
    std::size_t last_tokens() const { return last_tokens_; }
    const rf_clf_config& config() const { return cfg_; }

private:
    rf_clf_config cfg_;
    std::size_t max_tokens_;
    rf_clf* clf_ = nullptr;
    mutable std::mutex mu_;
    mutable std::size_t last_tokens_ = 0;
};

inline std::vector<double> softmax(const std::vector<float>& z) {
    double m = -1e300, s = 0.0;
    for (float v : z) m = std::max(m, static_cast<double>(v));
    std::vector<double> p(z.size());
    for (std::size_t i = 0; i < z.size(); ++i) s += (p[i] = std::exp(z[i] - m));
    for (auto& v : p) v /= s;
    return p;
}

// labels {benign, jailbreak}: score = P(jailbreak), flagged at the reference's default 0.5 boundary
class ModelJailbreakClassifier final : public JailbreakClassifier {
public:
    explicit ModelJailbreakClassifier(std::shared_ptr<const ModelSession> s, double threshold = 0.5) : s_(std::move(s)), threshold_(threshold) {
        if (s_->config().n_labels != 2) throw std::invalid_argument("jailbreak model needs 2 labels");
    }
    JailbreakSignal classify(std::string_view text) const override {
        const auto p = softmax(s_->logits(text));
        JailbreakSignal sig;
        sig.score = p[1];
        sig.flagged = sig.score >= threshold_;
        if (sig.flagged) sig.matched = "model";
        return sig;
    }

private:
    std::shared_ptr<const ModelSession> s_;
    double threshold_;
};

// one sigmoid per kind, in the reference's kind order (classifiers.hpp:21)
class ModelPiiClassifier final : public PiiClassifier {
public:
    explicit ModelPiiClassifier(std::shared_ptr<const ModelSession> s) : s_(std::move(s)) {
        if (s_->config().n_labels != 3) throw std::invalid_argument("PII model needs 3 labels");
    }
    PiiSignal classify(std::string_view text) const override {
        static const char* kKinds[3] = {"ssn", "email", "credit_card"};
        const auto z = s_->logits(text);
        PiiSignal sig;
        for (int i = 0; i < 3; ++i)
            if (z[i] > 0.0f) sig.kinds.emplace_back(kKinds[i]);
        sig.flagged = !sig.kinds.empty();
        return sig;
    }

private:
    std::shared_ptr<const ModelSession> s_;
};

class ModelDomainClassifier final : public DomainClassifier {
public:
    ModelDomainClassifier(std::shared_ptr<const ModelSession> s, std::vector<std::string> labels) : s_(std::move(s)), labels_(std::move(labels)) {
        if (static_cast<std::size_t>(s_->config().n_labels) != labels_.size()) throw std::invalid_argument("domain model: label count mismatch");
    }
    DomainSignal classify(std::string_view text) const override {
        const auto p = softmax(s_->logits(text));
        const std::size_t k = static_cast<std::size_t>(std::max_element(p.begin(), p.end()) - p.begin());
        DomainSignal sig;
        sig.label = labels_[k];
        sig.score = p[k];
        return sig;
    }

private:
    std::shared_ptr<const ModelSession> s_;
    std::vector<std::string> labels_;
};

struct ClassifierSet {  // classifiers.hpp:74-80
    std::shared_ptr<const JailbreakClassifier> jailbreak;
    std::shared_ptr<const PiiClassifier> pii;
    std::shared_ptr<const DomainClassifier> domain;

    // Three model-backed classifiers (safety, PII, domain: BASELINE config 3) with random-init weights from
    // distinct seeds, all sharing `base` except for the label count.
    static ClassifierSet model_backed(rf_clf_config base, std::vector<std::string> domains, int device = 0, uint64_t seed = 7,
                                      double jailbreak_threshold = 0.5) {
        auto make = [&](int n_labels, uint64_t sd) {
            rf_clf_config c = base;
            c.n_labels = n_labels;
            return std::make_shared<const ModelSession>(c, random_init_weights(c, sd), device);
        };
        ClassifierSet set;
        set.jailbreak = std::make_shared<const ModelJailbreakClassifier>(make(2, seed), jailbreak_threshold);
        set.pii = std::make_shared<const ModelPiiClassifier>(make(3, seed + 1));
        set.domain = std::make_shared<const ModelDomainClassifier>(make(static_cast<int>(domains.size()), seed + 2), std::move(domains));
        return set;
    }
};

}  // namespace routefast_b200
