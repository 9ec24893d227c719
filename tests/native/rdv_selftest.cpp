// Host-rendezvous self-test (CPU): the DD_COMM_IPC shared-memory rendezvous
// across forked processes and the DD_COMM_LOCAL one across threads --
// allgather contents, many back-to-back rounds (slot double-buffering), and a
// missing rank -> every waiting rank fails after the timeout (no hang).
// Built and run by tests/test_rendezvous_host.py; includes comm.cpp so the
// internal classes are reachable (the rest resolves against libdd.so).
#include "../../paper_2508_04917_b200/csrc/comm.cpp"

#include <sys/wait.h>

#include <cstdio>
#include <thread>

using namespace ddi;

static int run_rank(Rendezvous *R, int world, int rank, int rounds) {
    for (int it = 0; it < rounds; ++it) {
        int64_t mine[3] = {rank, it, 1000 * rank + it};
        std::vector<uint8_t> all;
        if (!R->allgather(mine, sizeof mine, all)) return 10;
        if (all.size() != sizeof mine * world) return 11;
        for (int q = 0; q < world; ++q) {
            int64_t v[3];
            std::memcpy(v, &all[q * sizeof v], sizeof v);
            if (v[0] != q || v[1] != it || v[2] != 1000 * q + it) return 12;
        }
    }
    return 0;
}

int main(int argc, char **argv) {
    const std::string mode = argc > 1 ? argv[1] : "shm";
    const int world = argc > 2 ? atoi(argv[2]) : 3;
    uint8_t key[128];
    for (int q = 0; q < 128; ++q) key[q] = (uint8_t)(rand() ^ getpid() ^ (q * 131));
    if (mode == "shm" || mode == "shm_missing") {
        const int present = mode == "shm" ? world : world - 1;
        std::vector<pid_t> kids;
        for (int r = 0; r < present; ++r) {
            const pid_t p = fork();
            if (p == 0) {
                ShmRdv *R = ShmRdv::join(key, world, r);
                if (!R) _exit(20);
                int rc = run_rank(R, world, r, mode == "shm" ? 200 : 1);
                if (mode == "shm" && rc == 0) R->setup_done();
                delete R;
                _exit(rc);
            }
            kids.push_back(p);
        }
        int bad = 0;
        for (pid_t p : kids) {
            int st = 0;
            waitpid(p, &st, 0);
            const int rc = WIFEXITED(st) ? WEXITSTATUS(st) : 99;
            if (mode == "shm" ? rc != 0 : rc != 10) bad = rc ? rc : 1;
        }
        printf("%s world %d: %s\n", mode.c_str(), world, bad ? "FAIL" : "ok");
        return bad;
    }
    // local: threads
    const int present = mode == "local" ? world : world - 1;
    std::vector<int> rcs(present, -1);
    std::vector<std::thread> th;
    for (int r = 0; r < present; ++r)
        th.emplace_back([&, r] {
            Rendezvous *R = local_join(key, world, r);
            rcs[r] = R ? run_rank(R, world, r, mode == "local" ? 200 : 1) : 20;
            delete R;
        });
    for (auto &t : th) t.join();
    int bad = 0;
    for (int rc : rcs)
        if (mode == "local" ? rc != 0 : rc != 10) bad = rc ? rc : 1;
    printf("%s world %d: %s\n", mode.c_str(), world, bad ? "FAIL" : "ok");
    return bad;
}
