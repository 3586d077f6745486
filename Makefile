# Build of the B200-native SpTTN engine (invoked by __graft_entry__.build()).
#
#   lib/libspttn_b200.so       CUDA kernels + C-ABI (include/spttn_b200.h), sm_100a
#   lib/libspttn_datagen.so    host synthetic-tensor generators / COO->CSF
#   lib/libspttn_b200_host.so  C++ shim: spttn::prepare/execute/... over the C-ABI,
#                              linked with the reference's host planner
#                              (built from /root/reference when present)
#   build/tests/*              C++ parity / acceptance binaries against the shim
#   oracle/                    test-only oracle builds (oracle/Makefile)
NVCC      ?= nvcc
CXX       ?= g++
PKG       := paper_2307_05740_b200
LIB       := $(PKG)/lib
DEV_SRC   := $(wildcard $(PKG)/csrc/device/*.cu)
DEV_HDR   := $(wildcard $(PKG)/csrc/device/*.cuh) $(PKG)/csrc/device/program.h include/spttn_b200.h
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -warn-spills
REF       ?= /root/reference/proj
PLANNER   := tensor kernel_spec contraction_path loop_nest cost_model optimizer tns_io bench
PLAN_OBJS := $(addprefix build/planner/,$(addsuffix .o,$(PLANNER)))
HOSTFLAGS := -std=c++20 -O2 -fPIC -I$(REF)/include -Iinclude -I$(PKG)/csrc/device

DEV_OBJS  := $(patsubst $(PKG)/csrc/device/%.cu,build/device/%.o,$(DEV_SRC))

all: device debug datagen probe oracle host
device: $(LIB)/libspttn_b200.so
# bounds-checked engine (device SPTTN_DCHECKs; SPTTN_DEBUG_BOUNDS=1 loads it)
debug: $(LIB)/debug/libspttn_b200.so
probe: $(LIB)/libspttn_probe.so
datagen: $(LIB)/libspttn_datagen.so
HAVE_HOST := $(and $(wildcard $(REF)/src/loop_nest.cpp),$(wildcard $(PKG)/csrc/shim/executor_b200.cpp))
ifneq ($(HAVE_HOST),)
host: $(LIB)/libspttn_b200_host.so build/tests/test_executor_b200 build/tests/acceptance_b200 build/tests/plan_overhead build/tests/generic_scale
else
host:
	@echo "reference sources absent: keeping prebuilt host shim"
endif

build/device/%.o: $(PKG)/csrc/device/%.cu $(DEV_HDR)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@

# the forest interpreter follows the reference's host arithmetic exactly
# (separate multiply and add): no FMA contraction in this file
build/device/generic.o: $(PKG)/csrc/device/generic.cu $(DEV_HDR)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -fmad=false -c $< -o $@

$(LIB)/libspttn_b200.so: $(DEV_OBJS)
	@mkdir -p $(LIB)
	$(NVCC) $(ARCH) -shared $^ -o $@ -lnvrtc -Xlinker -rpath,/usr/local/cuda/lib64

DBG_OBJS  := $(patsubst $(PKG)/csrc/device/%.cu,build/device_dbg/%.o,$(DEV_SRC))
build/device_dbg/%.o: $(PKG)/csrc/device/%.cu $(DEV_HDR)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -DSPTTN_DEBUG_BOUNDS -c $< -o $@
build/device_dbg/generic.o: $(PKG)/csrc/device/generic.cu $(DEV_HDR)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -DSPTTN_DEBUG_BOUNDS -fmad=false -c $< -o $@
$(LIB)/debug/libspttn_b200.so: $(DBG_OBJS)
	@mkdir -p $(LIB)/debug
	$(NVCC) $(ARCH) -shared $^ -o $@ -lnvrtc -Xlinker -rpath,/usr/local/cuda/lib64

$(LIB)/libspttn_probe.so: $(PKG)/csrc/probe/fp64_peak.cu
	@mkdir -p $(LIB)
	$(NVCC) $(NVFLAGS) -shared $< -o $@

$(LIB)/libspttn_datagen.so: $(PKG)/csrc/host/datagen.cpp
	@mkdir -p $(LIB)
	$(CXX) -std=c++17 -O3 -fPIC -shared $< -o $@

# The reference's host planner (path enumeration, loop-order DP, cost models,
# forest construction) — kept running on the host per the north star; the
# executor.cpp it normally links with is replaced by our shim.
build/planner/%.o: $(REF)/src/%.cpp
	@mkdir -p $(dir $@)
	$(CXX) $(HOSTFLAGS) -c $< -o $@

build/shim/executor_b200.o: $(PKG)/csrc/shim/executor_b200.cpp $(PKG)/csrc/device/program.h include/spttn_b200.h
	@mkdir -p $(dir $@)
	$(CXX) $(HOSTFLAGS) -c $< -o $@

$(LIB)/libspttn_b200_host.so: build/shim/executor_b200.o $(PLAN_OBJS) $(LIB)/libspttn_b200.so
	$(CXX) -shared build/shim/executor_b200.o $(PLAN_OBJS) -L$(LIB) -lspttn_b200 \
	  -Wl,-rpath,'$$ORIGIN' -o $@

build/tests/test_executor_b200: tests/cpp/test_executor_b200.cpp $(LIB)/libspttn_b200_host.so
	@mkdir -p $(dir $@)
	$(CXX) $(HOSTFLAGS) -I$(REF)/tests $< -L$(LIB) -lspttn_b200_host -lspttn_b200 \
	  -Wl,-rpath,'$$ORIGIN/../../$(LIB)' -o $@

# The reference's own acceptance harness linked against the device executor.
build/tests/acceptance_b200: $(REF)/tests/acceptance.cpp $(LIB)/libspttn_b200_host.so
	@mkdir -p $(dir $@)
	$(CXX) $(HOSTFLAGS) -I$(REF)/tests $< -L$(LIB) -lspttn_b200_host -lspttn_b200 \
	  -Wl,-rpath,'$$ORIGIN/../../$(LIB)' -o $@

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all device debug datagen probe host oracle clean

build/tests/plan_overhead: tests/cpp/plan_overhead.cpp $(LIB)/libspttn_b200_host.so
	@mkdir -p $(dir $@)
	$(CXX) $(HOSTFLAGS) -I$(REF)/tests $< -L$(LIB) -lspttn_b200_host -lspttn_b200 \
	  -Wl,-rpath,'$$ORIGIN/../../$(LIB)' -o $@

build/tests/generic_scale: tests/cpp/generic_scale.cpp $(LIB)/libspttn_b200_host.so
	@mkdir -p $(dir $@)
	$(CXX) $(HOSTFLAGS) -I$(REF)/tests $< -L$(LIB) -lspttn_b200_host -lspttn_b200 \
	  -Wl,-rpath,'$$ORIGIN/../../$(LIB)' -o $@

# Microbenchmark probes behind the DESIGN.md measurements (not part of `all`;
# binaries are git-ignored): make probes
PROBES := $(patsubst tools/%.cu,tools/%,$(wildcard tools/*_probe.cu))
probes: $(PROBES)
tools/%_probe: tools/%_probe.cu
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 $< -o $@ -lcuda
.PHONY: probes

# Drop-in pinned to the reference executor in one process: the reference side
# is compiled with -Dspttn=spttn_ref and linked with oracle/_ref/libspttn_ref.a
# (oracle/Makefile), the drop-in side with libspttn_b200_host.so.
REF_LIB := oracle/_ref/libspttn_ref.a
ifneq ($(HAVE_HOST),)
host: build/tests/ref_pin
endif
build/tests/ref_side.o: tests/cpp/ref_side.cpp tests/cpp/ref_side.hpp
	@mkdir -p $(dir $@)
	$(CXX) -std=c++20 -O2 -fPIC -Dspttn=spttn_ref -I$(REF)/include -I$(REF)/tests -c $< -o $@
build/tests/ref_pin: tests/cpp/ref_pin.cpp build/tests/ref_side.o $(LIB)/libspttn_b200_host.so oracle
	$(CXX) $(HOSTFLAGS) -I$(REF)/tests -Itests/cpp $< build/tests/ref_side.o $(REF_LIB) \
	  -L$(LIB) -lspttn_b200_host -lspttn_b200 -Wl,-rpath,'$$ORIGIN/../../$(LIB)' -o $@
