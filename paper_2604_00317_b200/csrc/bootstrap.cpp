// TCP rendezvous; see bootstrap.hpp.
#include "bootstrap.hpp"

#include <arpa/inet.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <poll.h>
#include <sys/mman.h>
#include <sys/socket.h>
#include <fcntl.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>

#include "capi_util.hpp"

namespace nb {

namespace {

constexpr uint32_t kMagic = 0x4e4d4231;  // "NMB1"
// a silent peer for 10 min is dead (NIMBLE_BOOTSTRAP_TIMEOUT_MS overrides)
int io_timeout_ms() {
    static const int ms = [] {
        const char* e = std::getenv("NIMBLE_BOOTSTRAP_TIMEOUT_MS");
        const int v = e && *e ? std::atoi(e) : 0;
        return v > 0 ? v : 600000;
    }();
    return ms;
}

struct IdBlob {
    uint32_t magic;
    uint32_t addr;  // IPv4, network order
    uint16_t port;  // network order
    uint16_t pad;
    uint64_t nonce;
};
static_assert(sizeof(IdBlob) <= NIMBLE_UNIQUE_ID_BYTES, "id blob too large");

struct Hello {
    uint32_t magic;
    int32_t rank, nranks;
    uint32_t pad;
    uint64_t nonce;
};

[[noreturn]] void sys_fail(const std::string& what) {
    throw Error(nimbleSystemError, "bootstrap: " + what + ": " + std::strerror(errno));
}

void wait_io(int fd, short ev) {
    pollfd p{fd, ev, 0};
    int r = ::poll(&p, 1, io_timeout_ms());
    if (r == 0) throw Error(nimbleRemoteError, "bootstrap: peer timed out");
    if (r < 0 && errno != EINTR) sys_fail("poll");
}

void send_all(int fd, const void* p, size_t n) {
    auto* b = static_cast<const uint8_t*>(p);
    while (n) {
        wait_io(fd, POLLOUT);
        ssize_t k = ::send(fd, b, n, MSG_NOSIGNAL);
        if (k < 0) {
            if (errno == EINTR || errno == EAGAIN) continue;
            sys_fail("send");
        }
        b += k;
        n -= static_cast<size_t>(k);
    }
}

// false on orderly close before any byte
bool recv_all(int fd, void* p, size_t n) {
    auto* b = static_cast<uint8_t*>(p);
    size_t got = 0;
    while (got < n) {
        wait_io(fd, POLLIN);
        ssize_t k = ::recv(fd, b + got, n - got, 0);
        if (k == 0) {
            if (got == 0) return false;
            throw Error(nimbleRemoteError, "bootstrap: peer closed mid-message");
        }
        if (k < 0) {
            if (errno == EINTR || errno == EAGAIN) continue;
            sys_fail("recv");
        }
        got += static_cast<size_t>(k);
    }
    return true;
}

void tune(int fd) {
    int one = 1;
    ::setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &one, sizeof one);
}

// Root service: accept nranks members, then run allgather rounds until every
// member has closed its socket.
void serve(int lfd, uint64_t nonce) {
    std::vector<int> fds;
    try {
        int nranks = -1;
        std::vector<std::pair<int, int>> joined;  // (rank, fd)
        while (nranks < 0 || static_cast<int>(joined.size()) < nranks) {
            wait_io(lfd, POLLIN);
            int fd = ::accept(lfd, nullptr, nullptr);
            if (fd < 0) {
                if (errno == EINTR) continue;
                sys_fail("accept");
            }
            tune(fd);
            Hello h{};
            if (!recv_all(fd, &h, sizeof h) || h.magic != kMagic || h.nonce != nonce) {
                ::close(fd);
                continue;
            }
            if (nranks < 0) nranks = h.nranks;
            if (h.nranks != nranks || h.rank < 0 || h.rank >= nranks) {
                ::close(fd);
                continue;
            }
            joined.push_back({h.rank, fd});
        }
        fds.assign(static_cast<size_t>(nranks), -1);
        for (auto& [r, fd] : joined) fds[static_cast<size_t>(r)] = fd;
        for (int fd : fds)
            if (fd < 0) throw Error(nimbleInternalError, "bootstrap: duplicate rank");
        for (;;) {
            std::vector<uint8_t> all;
            uint64_t n = 0;
            bool closed = false;
            for (size_t r = 0; r < fds.size(); ++r) {
                uint64_t len = 0;
                if (!recv_all(fds[r], &len, sizeof len)) {
                    closed = true;
                    break;
                }
                if (r == 0) {
                    n = len;
                    all.resize(n * fds.size());
                } else if (len != n) {
                    throw Error(nimbleInvalidUsage, "bootstrap: allgather sizes differ across ranks");
                }
                if (n && !recv_all(fds[r], all.data() + r * n, n))
                    throw Error(nimbleRemoteError, "bootstrap: short allgather");
            }
            if (closed) break;
            for (int fd : fds) send_all(fd, all.data(), all.size());
        }
    } catch (...) {
    }
    for (int fd : fds)
        if (fd >= 0) ::close(fd);
    ::close(lfd);
}

class TcpBootstrap final : public Bootstrap {
  public:
    TcpBootstrap(const IdBlob& id, int r, int n) {
        rank = r;
        nranks = n;
        sockaddr_in sa{};
        sa.sin_family = AF_INET;
        sa.sin_addr.s_addr = id.addr;
        sa.sin_port = id.port;
        const auto deadline = std::chrono::steady_clock::now() + std::chrono::seconds(120);
        for (;;) {
            fd_ = ::socket(AF_INET, SOCK_STREAM, 0);
            if (fd_ < 0) sys_fail("socket");
            if (::connect(fd_, reinterpret_cast<sockaddr*>(&sa), sizeof sa) == 0) break;
            ::close(fd_);
            fd_ = -1;
            if (std::chrono::steady_clock::now() > deadline)
                throw Error(nimbleRemoteError, "bootstrap: cannot reach the root");
            std::this_thread::sleep_for(std::chrono::milliseconds(20));
        }
        tune(fd_);
        Hello h{kMagic, r, n, 0, id.nonce};
        send_all(fd_, &h, sizeof h);
    }
    ~TcpBootstrap() override {
        if (fd_ >= 0) ::close(fd_);
    }
    void allgather(const void* mine, size_t n, void* all) override {
        uint64_t len = n;
        send_all(fd_, &len, sizeof len);
        if (n) send_all(fd_, mine, n);
        if (!recv_all(fd_, all, n * static_cast<size_t>(nranks)) && n)
            throw Error(nimbleRemoteError, "bootstrap: root closed");
    }

  private:
    int fd_ = -1;
};

}  // namespace

void bootstrap_root(nimbleUniqueId* id) {
    const char* env = std::getenv("NIMBLE_BOOTSTRAP_ADDR");
    in_addr addr{};
    if (::inet_pton(AF_INET, env && *env ? env : "127.0.0.1", &addr) != 1)
        throw Error(nimbleInvalidArgument, "bootstrap: bad NIMBLE_BOOTSTRAP_ADDR");
    int lfd = ::socket(AF_INET, SOCK_STREAM, 0);
    if (lfd < 0) sys_fail("socket");
    int one = 1;
    ::setsockopt(lfd, SOL_SOCKET, SO_REUSEADDR, &one, sizeof one);
    sockaddr_in sa{};
    sa.sin_family = AF_INET;
    sa.sin_addr = addr;
    sa.sin_port = 0;
    if (::bind(lfd, reinterpret_cast<sockaddr*>(&sa), sizeof sa) != 0) sys_fail("bind");
    if (::listen(lfd, 256) != 0) sys_fail("listen");
    socklen_t sl = sizeof sa;
    if (::getsockname(lfd, reinterpret_cast<sockaddr*>(&sa), &sl) != 0) sys_fail("getsockname");
    std::random_device rd;
    const uint64_t nonce = (static_cast<uint64_t>(rd()) << 32) ^ rd() ^ static_cast<uint64_t>(::getpid());
    IdBlob blob{kMagic, addr.s_addr, sa.sin_port, 0, nonce};
    std::memset(id, 0, sizeof *id);
    std::memcpy(id->internal, &blob, sizeof blob);
    std::thread(serve, lfd, nonce).detach();
}

// One rank's record, double-buffered by call parity: a writer can be at most
// one call ahead of the slowest reader (it cannot finish call k + 1 before
// every rank has written k + 1, i.e. finished reading k).
struct ShmAllgather::Slot {
    std::atomic<uint64_t> seq[2];
    uint8_t data[2][kRecord];
};

ShmAllgather::ShmAllgather(const nimbleUniqueId& id, Bootstrap& boot) : rank_(boot.rank), nranks_(boot.nranks) {
    IdBlob blob;
    std::memcpy(&blob, id.internal, sizeof blob);
    char name[64];
    std::snprintf(name, sizeof name, "/nimble-%016llx-%04x", static_cast<unsigned long long>(blob.nonce),
                  static_cast<unsigned>(blob.port));
    bytes_ = sizeof(Slot) * static_cast<size_t>(nranks_);
    if (rank_ == 0) {
        int fd = ::shm_open(name, O_CREAT | O_EXCL | O_RDWR, 0600);
        if (fd < 0) sys_fail("shm_open");
        if (::ftruncate(fd, static_cast<off_t>(bytes_)) != 0) {
            ::close(fd);
            ::shm_unlink(name);
            sys_fail("ftruncate");
        }
        ::close(fd);  // zero-filled: every seq starts at 0
    }
    boot.barrier();
    int fd = ::shm_open(name, O_RDWR, 0600);
    if (fd < 0) sys_fail("shm_open");
    void* p = ::mmap(nullptr, bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    ::close(fd);
    if (p == MAP_FAILED) sys_fail("mmap");
    slots_ = static_cast<Slot*>(p);
    boot.barrier();
    if (rank_ == 0) ::shm_unlink(name);  // the mappings stay; no file outlives the comm
}

ShmAllgather::~ShmAllgather() {
    if (slots_) ::munmap(slots_, bytes_);
}

void ShmAllgather::allgather(const void* mine, size_t n, void* all, uint32_t timeout_ms) {
    if (n > kRecord) throw Error(nimbleInternalError, "shm allgather: record too large");
    const uint64_t k = ++calls_;
    const int par = static_cast<int>(k & 1);
    Slot& me = slots_[rank_];
    std::memcpy(me.data[par], mine, n);
    me.seq[par].store(k, std::memory_order_release);
    const auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < nranks_; ++r) {
        Slot& s = slots_[r];
        for (uint32_t spin = 0; s.seq[par].load(std::memory_order_acquire) < k; ++spin) {
            if (spin > 1000) {
                std::this_thread::yield();
                if ((spin & 1023) == 0 &&
                    std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(timeout_ms))
                    throw Error(nimbleRemoteError, "shm allgather: a rank did not arrive");
            }
        }
        std::memcpy(static_cast<uint8_t*>(all) + static_cast<size_t>(r) * n, s.data[par], n);
    }
}

std::unique_ptr<Bootstrap> bootstrap_connect(const nimbleUniqueId& id, int rank, int nranks) {
    IdBlob blob;
    std::memcpy(&blob, id.internal, sizeof blob);
    if (blob.magic != kMagic) throw Error(nimbleInvalidArgument, "bootstrap: not a nimble unique id");
    if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(nimbleInvalidArgument, "bootstrap: bad rank");
    return std::make_unique<TcpBootstrap>(blob, rank, nranks);
}

}  // namespace nb
