// protocol_test.cpp -- the reference's bench_test.cpp / io scenarios on the
// GPU-backed C++ mirror: seed-0 draw pins, the 20-trial golden CSV (counter
// columns, time columns stripped), aggregate formats, text fixture round trip.
#include <mh/mh.hpp>

#include <cstdio>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

namespace {
int g_checks = 0, g_fail = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        ++g_checks;                                                           \
        if (!(c)) {                                                           \
            ++g_fail;                                                         \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
        }                                                                     \
    } while (0)

std::string slurp(const std::string& p) {
    std::ifstream is(p);
    std::stringstream ss;
    ss << is.rdbuf();
    return ss.str();
}

std::string strip_two(const std::string& csv) {
    std::stringstream in(csv), out;
    std::string line;
    while (std::getline(in, line)) {
        std::size_t end = line.size();
        for (int k = 0; k < 2; ++k) end = line.rfind(',', end - 1);
        out << line.substr(0, end) << '\n';
    }
    return out.str();
}
}  // namespace

// layout_test.cpp:147-175: the text format round-trips and is exact; malformed files
// raise std::invalid_argument
void io_cases() {
    std::mt19937_64 eng(11);
    mh::Grid g(8, std::vector<mh::Fp>(8));
    for (auto& row : g)
        for (auto& c : row) c = mh::Fp{std::uint32_t(eng() % 97)};
    const mh::Matrix m = mh::from_row_major(g, 4, mh::Modulus(97));
    std::ostringstream os;
    mh::save_matrix(os, m);
    const std::string text = os.str();
    CHECK(text.substr(0, 7) == "8 4 97\n");
    CHECK(text.back() == '\n');
    std::istringstream is(text);
    CHECK(mh::load_matrix(is) == m);
    auto rejects = [](const std::string& s) {
        std::istringstream in(s);
        try {
            (void)mh::load_matrix(in);
        } catch (const std::invalid_argument&) {
            return true;
        } catch (...) {
            return false;
        }
        return false;
    };
    CHECK(rejects(""));
    CHECK(rejects("2 1\n0 0\n0 0\n"));    // truncated header
    CHECK(rejects("2 1 4\n0 0\n0 0\n"));  // composite modulus
    CHECK(rejects("2 1 2\n0 0\n0\n"));    // missing residue
    CHECK(rejects("2 1 2\n0 0\n0 2\n"));  // residue >= q
    CHECK(rejects("2 1 2\n0 0\n0 -1\n"));
    CHECK(rejects("6 3 2\n"));              // 6 / 3 is not a power of two
}

int main(int argc, char** argv) {
    // --save n t q seed path: a container filled from mh::Rng(seed) in flat Morton
    // order, written by save_matrix_file (byte parity with the reference's writer is
    // checked by tests/test_cpp_dropin.py)
    if (argc == 7 && std::string(argv[1]) == "--save") {
        const std::uint64_t n = std::stoull(argv[2]), t = std::stoull(argv[3]);
        const std::uint32_t q = (std::uint32_t)std::stoul(argv[4]);
        mh::Rng rng(std::stoull(argv[5]));
        mh::Matrix m(mh::Layout(n, t), mh::Modulus(q));
        for (auto& v : m.cells()) v = mh::Fp{std::uint32_t(rng.below(q))};
        mh::save_matrix_file(argv[6], m);
        const mh::Matrix back = mh::load_matrix_file(argv[6]);
        return back == m ? 0 : 1;
    }
    const std::string golden_path = argc > 1 ? argv[1] : "tests/golden/bench_trials_seed0_n64_t8_q2.csv";
    io_cases();
    mh::Config cfg;
    cfg.n = 64;
    cfg.t = 8;
    cfg.q = 2;
    cfg.seed = 0;
    {  // bench_test.cpp:56-72
        mh::Rng rng(0);
        const auto inst = mh::gen_problem(cfg, rng);
        CHECK(inst.sa.origin == 1 && inst.sa.rows == 64 && inst.sa.cols == 39);
        CHECK(inst.sb.origin == 322 && inst.sb.cols == 3 && inst.sc.origin == 2855);
        CHECK(!inst.aligned_draw);
        unsigned long long h = 0;
        for (mh::Index z = 0; z < inst.a->layout().total; ++z) h = h * 31 + (*inst.a)[z].v;
        CHECK(h == 4715125990397575263ull);
    }
    {  // bench_test.cpp:74-115 on the GPU engine
        cfg.trials = 20;
        const auto trials = mh::run_trials(cfg);
        CHECK(trials.size() == 20);
        mh::write_trials_csv(trials, "protocol_test_trials.csv");
        const std::string got = strip_two(slurp("protocol_test_trials.csv"));
        const std::string want = slurp(golden_path);
        CHECK(got == want);
        if (got != want) std::fprintf(stderr, "got:\n%s\nwant:\n%s\n", got.c_str(), want.c_str());
        const auto rows = mh::aggregate(trials);
        double share = 0;
        for (const auto& b : rows) share += b.share_pct;
        CHECK(share > 99.9 && share < 100.1);
        mh::write_aggregate_csv(rows, "protocol_test_agg.csv");
        CHECK(slurp("protocol_test_agg.csv").rfind(mh::kAggregateCsvHeader, 0) == 0);
        std::remove("protocol_test_trials.csv");
        std::remove("protocol_test_agg.csv");
    }
    {  // config validation, bench_test.cpp:118-131
        mh::Config bad = cfg;
        bad.t = 7;
        bool threw = false;
        try { mh::check_config(bad); } catch (const std::invalid_argument&) { threw = true; }
        CHECK(threw);
    }
    {  // io.hpp round trip through the device conversion kernels
        mh::Rng rng(3);
        mh::Matrix m(mh::Layout(24, 3), mh::Modulus(97));
        for (auto& v : m.cells()) v = mh::Fp{std::uint32_t(rng.below(97))};
        std::stringstream ss;
        mh::save_matrix(ss, m);
        const mh::Matrix back = mh::load_matrix(ss);
        CHECK(back == m);
        std::stringstream bad("8 4 97\n1 2 3\n");
        bool threw = false;
        try { mh::load_matrix(bad); } catch (const std::invalid_argument&) { threw = true; }
        CHECK(threw);
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
