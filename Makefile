# Build of the B200 linear-recurrence library (in-tree; the .so files travel
# to the GPU box with the gpurun snapshot).
#
#   make            liblinrec_cuda.so (C ABI) + the `linrec` Python module +
#                   the CPU oracle (test infrastructure)
#   make ref        also compile the reference from /root/reference into
#                   oracle/_ref (only where /root/reference exists)
#
# sm_100a only: no other architectures, no PTX fallback.

PY      ?= python3
NVCC    ?= /usr/local/cuda/bin/nvcc
# the image exports CXX=/opt/gcc/bin/g++ (a wrapper with a different system
# include order); its -O2 build of the pybind module crashes on throw, so pin
# the distribution compiler.
CXX     := $(firstword $(wildcard /usr/bin/g++) g++)
PKG     := paper_1709_04057_b200
CSRC    := $(PKG)/csrc
BUILD   := build
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -std=c++17 -O3 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           -Iinclude -I$(CSRC) --expt-relaxed-constexpr
EXT     := $(shell $(PY) -c "import sysconfig;print(sysconfig.get_config_var('EXT_SUFFIX'))")
PYINC   := $(shell $(PY) -c "import pybind11,sysconfig;print('-I'+pybind11.get_include(),'-I'+sysconfig.get_paths()['include'])")

KERNEL_SRCS := $(CSRC)/chain_fwd_f32.cu $(CSRC)/chain_bwd_f32.cu $(CSRC)/chain_fwd_f64.cu \
               $(CSRC)/chain_bwd_f64.cu $(CSRC)/serial_misc.cu $(CSRC)/tma_fwd_f32.cu \
               $(CSRC)/tma_bwd_f32.cu $(CSRC)/tma_f64.cu $(CSRC)/segment.cu $(CSRC)/gemm_tc.cu \
               $(CSRC)/layers.cu $(CSRC)/layers_f64.cu $(CSRC)/training.cu $(CSRC)/p2p.cu $(CSRC)/plan_scan.cu $(CSRC)/local_scan.cu $(CSRC)/cluster_scan.cu
HOST_SRCS   := $(CSRC)/capi.cpp $(CSRC)/sharded_capi.cpp
HDRS        := $(wildcard $(CSRC)/*.cuh) $(CSRC)/launch.h include/linrec_cuda.h
OBJS        := $(patsubst $(CSRC)/%.cu,$(BUILD)/%.o,$(KERNEL_SRCS)) $(BUILD)/capi.o $(BUILD)/sharded_capi.o

LIB   := $(PKG)/liblinrec_cuda.so
PYMOD := $(PKG)/linrec$(EXT)

CPPTEST := $(BUILD)/test_cuda_api
CPPSHARD := $(BUILD)/test_sharded

.PHONY: all lib py oracle ref clean cpp-tests
all: lib py oracle cpp-tests

# C++ caller of include/linrec/cuda_scan.hpp + cuda_layers.hpp (host code only:
# g++ against the C ABI and the CUDA runtime for device buffers).
cpp-tests: $(CPPTEST) $(CPPSHARD)
$(CPPSHARD): tests/cpp/test_sharded.cpp include/linrec/cuda_sharded.hpp include/linrec/cuda_scan.hpp include/linrec_cuda.h $(LIB)
	@mkdir -p $(BUILD)
	$(CXX) -std=c++17 -O2 -Iinclude -I/usr/local/cuda/include -o $@ $< -L$(PKG) -llinrec_cuda \
	  -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,'$$ORIGIN/../$(PKG)' -Wl,-rpath,/usr/local/cuda/lib64
$(CPPTEST): tests/cpp/test_cuda_api.cpp include/linrec/cuda_scan.hpp include/linrec/cuda_layers.hpp include/linrec/cuda_sharded.hpp include/linrec_cuda.h $(LIB)
	@mkdir -p $(BUILD)
	$(CXX) -std=c++17 -O2 -Iinclude -I/usr/local/cuda/include -o $@ $< -L$(PKG) -llinrec_cuda \
	  -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,'$$ORIGIN/../$(PKG)' -Wl,-rpath,/usr/local/cuda/lib64

lib: $(LIB)
py: $(PYMOD)

$(BUILD)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(BUILD)/capi.o: $(CSRC)/capi.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(BUILD)/sharded_capi.o: $(CSRC)/sharded_capi.cpp include/linrec_cuda.h
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

# Exported surface = the extern "C" functions of include/linrec_cuda.h
# (everything else is hidden).  cudart is linked statically.
$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS) -Xlinker --exclude-libs,ALL

$(PYMOD): $(CSRC)/linrec_py.cpp include/linrec/cuda_scan.hpp include/linrec_cuda.h $(LIB)
	$(CXX) -std=c++17 -O2 -fPIC -shared -fvisibility=hidden -Iinclude $(PYINC) \
	  -o $@ $(CSRC)/linrec_py.cpp -L$(PKG) -llinrec_cuda -Wl,-rpath,'$$ORIGIN'

oracle:
	$(MAKE) -C oracle PY=$(PY)

ref:
	$(MAKE) -C oracle ref PY=$(PY)

clean:
	rm -rf $(BUILD) $(LIB) $(PYMOD)
	$(MAKE) -C oracle clean
