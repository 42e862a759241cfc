// Developer probe: host load path phases (parse, completion, store build) on a
// program file. Build: g++ -std=c++20 -O2 -I paper_1909_01786_b200/csrc scripts/host_load_bench.cpp \
//   paper_1909_01786_b200/csrc/host/program.cpp paper_1909_01786_b200/csrc/host/compile.cpp -lpthread
#include <chrono>
#include <cstdio>
#include <fstream>
#include <sstream>

#include "host/compile.hpp"
#include "host/program.hpp"

int main(int argc, char** argv) {
    std::ifstream in(argv[1]);
    std::stringstream ss;
    ss << in.rdbuf();
    const std::string text = ss.str();
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    for (int rep = 0; rep < 3; ++rep) {
        const auto t0 = now();
        yas::Program p = yas::parse_text(text);
        const auto t1 = now();
        yas::Completion c = yas::compile_completion(p);
        const auto t2 = now();
        yas::StaticStore st = yas::build_store(c.nogoods, c.total_atoms);
        const auto t3 = now();
        std::printf("parse %.1f ms, completion %.1f ms (%zu nogoods), store %.1f ms (%u CSR, %zu lits)\n", ms(t0, t1),
                    ms(t1, t2), c.nogoods.size(), ms(t2, t3), st.size(), st.pool.size());
    }
}
