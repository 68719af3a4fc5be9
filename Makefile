# Top-level build: the product library (libcdx.so, sm_100a) and the test-only checkers.
#   make            -> paper_2412_20993_b200/lib/libcdx.so + oracle (liboracle.so, _ref/libcdxref.so)
#   make lib        -> libcdx.so only
#   make sass       -> SASS/resource dump of every kernel (profiles/sass_summary.txt)
NVCC    ?= /usr/local/cuda/bin/nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
# -fmad=false: no FMA contraction anywhere, so FP64 certaindex math rounds like the reference
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-O2 \
           -Xptxas -warn-spills --expt-relaxed-constexpr
PKG     := paper_2412_20993_b200
SRCS    := $(wildcard $(PKG)/csrc/*.cu) $(wildcard $(PKG)/csrc/*.cpp)
OBJS    := $(patsubst $(PKG)/csrc/%,build/obj/%.o,$(SRCS))
HDRS    := $(wildcard $(PKG)/csrc/*.cuh) include/cdx_c.h
LIB     := $(PKG)/lib/libcdx.so
# C++ host layer: the reference's C++ API (include/cdx/*.hpp) over the C-ABI
HOSTLIB := $(PKG)/lib/libcdxhost.so
HSRCS   := $(wildcard $(PKG)/csrc/host/*.cpp)
HOBJS   := $(patsubst $(PKG)/csrc/host/%.cpp,build/host/%.o,$(HSRCS))
HHDRS   := $(wildcard $(PKG)/csrc/host/*.hpp) include/cdx_c.h $(wildcard include/cdx/*.hpp)
HOSTCXX := g++
CXXFLAGS_HOST := -std=c++20 -O2 -fPIC -Wall -Wextra -Iinclude

DROPIN  := tests/cpp/bin/dropin_ours tests/cpp/bin/facade_latency_ours tests/cpp/bin/scheduler_cases tests/cpp/bin/batch_pipeline tests/cpp/bin/sim_cases \
           tests/cpp/bin/shard_world2

all: lib oracle dropin

lib: $(LIB) $(HOSTLIB)

build/host/%.o: $(PKG)/csrc/host/%.cpp $(HHDRS)
	@mkdir -p build/host
	$(HOSTCXX) $(CXXFLAGS_HOST) -c $< -o $@

$(HOSTLIB): $(HOBJS) $(LIB)
	$(HOSTCXX) -shared -o $@ $(HOBJS) -L$(PKG)/lib -lcdx -Wl,-rpath,'$$ORIGIN'

build/obj/%.cu.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -Iinclude -c $< -o $@

build/obj/%.cpp.o: $(PKG)/csrc/%.cpp $(HDRS)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -Iinclude -x cu -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lpthread -ldl

oracle:
	$(MAKE) -C oracle

# drop-in proof: the same caller source the oracle builds against the reference headers
dropin: $(DROPIN)

CPPTEST = @mkdir -p tests/cpp/bin && $(HOSTCXX) -std=c++20 -O2 -Wall -Iinclude -o $@ $< -L$(PKG)/lib -lcdxhost -lcdx \
          -Wl,-rpath,'$$ORIGIN/../../../$(PKG)/lib'
tests/cpp/bin/dropin_ours: tests/cpp/dropin_cases.cpp $(HOSTLIB) $(HHDRS)
	$(CPPTEST)
tests/cpp/bin/facade_latency_ours: tests/cpp/facade_latency.cpp $(HOSTLIB) $(HHDRS)
	$(CPPTEST)
# multi-rank C-ABI test: W host threads, one context each, host-staged communicator callbacks
tests/cpp/bin/shard_world2: tests/cpp/shard_world2.cpp $(LIB) include/cdx_c.h
	@mkdir -p tests/cpp/bin && $(HOSTCXX) -std=c++20 -O2 -Wall -Iinclude -I/usr/local/cuda/include -o $@ $< \
	  -L$(PKG)/lib -lcdx -L/usr/local/cuda/lib64 -lcudart -lpthread \
	  -Wl,-rpath,'$$ORIGIN/../../../$(PKG)/lib' -Wl,-rpath,/usr/local/cuda/lib64
tests/cpp/bin/%: tests/cpp/%.cpp $(HOSTLIB) $(HHDRS)
	$(CPPTEST)

sass: $(LIB)
	@mkdir -p profiles
	/usr/local/cuda/bin/cuobjdump -res-usage $(LIB) > profiles/sass_resources.txt 2>&1 || true

clean:
	rm -rf build $(PKG)/lib tests/cpp/bin
	$(MAKE) -C oracle clean

.PHONY: all lib oracle dropin sass clean
