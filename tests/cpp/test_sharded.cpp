// One rank of the sequence-sharded scan driven from C++ through
// include/linrec/cuda_sharded.hpp (the multi-GPU C ABI): no Python, no
// torch.distributed.  tests/test_gpu_cpp_api.py starts `world` of these
// processes (sharing the test box's GPU, so the "NVLink" peers are CUDA-IPC
// mappings on one device); they exchange their 64-byte mailbox handles
// through files in <dir>, run <steps> forward + backward steps on their rows
// of the [T][W] problem in <dir>/{lam,x,h0,dh}.bin and write their rows of
// h, dlam, dx (+ dh0 on rank 0) to <dir>/out_<rank>_*.bin for the oracle
// comparison on the Python side.
//
//   test_sharded <dir> <rank> <world> <T> <W> <steps>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <thread>
#include <vector>

#include "linrec/cuda_sharded.hpp"

using namespace linrec::cuda;

static std::vector<float> read_rows(const std::string& path, size_t first, size_t count) {
  std::vector<float> v(count);
  std::ifstream f(path, std::ios::binary);
  f.seekg(std::streamoff(first * 4));
  f.read(reinterpret_cast<char*>(v.data()), std::streamsize(count * 4));
  if (!f) {
    std::fprintf(stderr, "read %s failed\n", path.c_str());
    std::exit(3);
  }
  return v;
}

static void write_all(const std::string& path, const float* d, size_t count) {
  std::vector<float> v(count);
  cudaMemcpy(v.data(), d, count * 4, cudaMemcpyDeviceToHost);
  const std::string tmp = path + ".tmp";
  std::ofstream(tmp, std::ios::binary).write(reinterpret_cast<const char*>(v.data()), std::streamsize(count * 4));
  std::rename(tmp.c_str(), path.c_str());
}

static float* upload(const std::vector<float>& v) {
  float* d = nullptr;
  if (cudaMalloc(&d, v.size() * 4 + 16) != cudaSuccess) std::abort();
  cudaMemcpy(d, v.data(), v.size() * 4, cudaMemcpyHostToDevice);
  return d;
}

int main(int argc, char** argv) {
  if (argc != 7) {
    std::fprintf(stderr, "usage: %s dir rank world T W steps\n", argv[0]);
    return 2;
  }
  const std::string dir = argv[1];
  const int rank = std::atoi(argv[2]), world = std::atoi(argv[3]);
  const index_t T = std::atoll(argv[4]), W = std::atoll(argv[5]);
  const int steps = std::atoi(argv[6]);
  try {
    cudaSetDevice(0);
    PeerMailbox mb(W, world, rank);
    {  // publish this rank's handle, then collect everyone's
      const std::string p = dir + "/handle_" + std::to_string(rank);
      std::ofstream(p + ".tmp", std::ios::binary)
          .write(reinterpret_cast<const char*>(mb.handle().data()), std::streamsize(mb.handle().size()));
      std::rename((p + ".tmp").c_str(), p.c_str());
    }
    std::vector<PeerMailbox::Handle> handles(static_cast<size_t>(world));
    for (int q = 0; q < world; ++q) {
      const std::string p = dir + "/handle_" + std::to_string(q);
      for (int tries = 0;; ++tries) {
        std::ifstream f(p, std::ios::binary);
        if (f && f.read(reinterpret_cast<char*>(handles[size_t(q)].data()), 64)) break;
        if (tries > 6000) throw std::runtime_error("timed out waiting for " + p);
        std::this_thread::sleep_for(std::chrono::milliseconds(10));
      }
    }
    mb.open(handles);
    SequenceShardedScan run(T, W, world, rank, mb, 0);
    const auto [r0, n] = run.rows();
    const auto sh = shard_rows(T, world, rank);
    if (sh.first != r0 || sh.second != n) throw std::runtime_error("shard_rows disagrees with the context");
    float* lam = upload(read_rows(dir + "/lam.bin", size_t(r0 * W), size_t(n * W)));
    float* x = upload(read_rows(dir + "/x.bin", size_t(r0 * W), size_t(n * W)));
    float* dh = upload(read_rows(dir + "/dh.bin", size_t(r0 * W), size_t(n * W)));
    float* h0 = upload(read_rows(dir + "/h0.bin", 0, size_t(W)));
    float *h, *dlam, *dx, *dh0;
    cudaMalloc(&h, size_t(n * W) * 4 + 16);
    cudaMalloc(&dlam, size_t(n * W) * 4 + 16);
    cudaMalloc(&dx, size_t(n * W) * 4 + 16);
    cudaMalloc(&dh0, size_t(W) * 4 + 16);
    const index_t b = 1;
    DeviceTensor3<float> tl{lam, n, b, W}, tx{x, n, b, W}, th{h, n, b, W}, tdh{dh, n, b, W};
    DeviceTensor2<float> t0{h0, b, W};
    RecurrenceGradients<float> g{{dlam, n, b, W}, {dx, n, b, W}, {dh0, b, W}};
    cudaStream_t st;
    cudaStreamCreate(&st);
    for (int s = 0; s < steps; ++s) {  // repeated steps reuse the mailboxes (epochs, acks)
      run.scan(tl, tx, t0, th, st);
      run.scan_backward(tl, t0, th, tdh, g, st);
    }
    if (cudaStreamSynchronize(st) != cudaSuccess) throw std::runtime_error("stream failed");
    const std::string o = dir + "/out_" + std::to_string(rank) + "_";
    write_all(o + "h.bin", h, size_t(n * W));
    write_all(o + "dlam.bin", dlam, size_t(n * W));
    write_all(o + "dx.bin", dx, size_t(n * W));
    if (rank == 0) write_all(o + "dh0.bin", dh0, size_t(W));
    // keep this rank's mailbox alive until every peer is done with it
    std::ofstream(dir + "/done_" + std::to_string(rank)) << "ok";
    for (int q = 0; q < world; ++q)
      for (int tries = 0; !std::ifstream(dir + "/done_" + std::to_string(q)); ++tries) {
        if (tries > 6000) throw std::runtime_error("timed out waiting for peers to finish");
        std::this_thread::sleep_for(std::chrono::milliseconds(10));
      }
    std::printf("rank %d rows [%lld, %lld) OK\n", rank, (long long)r0, (long long)(r0 + n));
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "rank %d: %s\n", rank, e.what());
    return 1;
  }
}
