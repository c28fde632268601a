"""The README's usage example, runnable: python tools/readme_example.py (needs a GPU)."""
import sys; import os; sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..'))
import torch, paper_2111_08692_b200 as ug
t8 = torch.frombuffer(bytearray("héllo, wörld ✓ 😀".encode()), dtype=torch.uint8).cuda()
n16 = ug.utf16_length_from_utf8(t8)
u16 = torch.empty(n16, dtype=torch.int16, device="cuda")
r = ug.utf8_to_utf16le(t8, u16)
print(r, n16, r.error == ug.OK, r.written == n16)
r2, n = ug.utf8_to_utf16le_two_pass(t8, u16)
print(r2, n)
print(u16.cpu().numpy().view('uint16').tobytes().decode('utf-16-le'))
